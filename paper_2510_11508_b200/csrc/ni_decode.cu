// Decode of 16-bit PNG normal maps (fileio.py:134-161) on the GPU: the host
// only inflates the PNG (cv2); the uint16 BGR samples (6 B/px instead of
// 24 B/px of float64) go to the device, where v / 65535 * 2 - 1, the norm
// sqrt((x^2 + y^2) + z^2) and the division reproduce numpy's float64
// arithmetic operation by operation (no FMA contraction).
#include "ni_common.cuh"

namespace ni {

__global__ void decode_png16_kernel(const uint16_t* __restrict__ bgr, int64_t npix, int flip_z,
                                    double* __restrict__ n_out, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint16_t b = bgr[3 * i], g = bgr[3 * i + 1], r = bgr[3 * i + 2];
    bool m = (r | g | b) != 0;
    double v[3] = {double(r), double(g), double(b)};  // rgb = img[..., ::-1]
#pragma unroll
    for (int c = 0; c < 3; ++c) v[c] = __dsub_rn(__dmul_rn(__ddiv_rn(v[c], 65535.0), 2.0), 1.0);
    if (flip_z) v[2] = -v[2];
    const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                           __dmul_rn(v[2], v[2])));
    m = m && nn > 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) n_out[3 * i + c] = m ? __ddiv_rn(v[c], nn) : 0.0;
    mask[i] = m;
  }
}

}  // namespace ni

using namespace ni;

extern "C" int ni_decode_png16(const uint16_t* bgr, int H, int W, int flip_z, double* n_out,
                               uint8_t* mask_out, ni_stream_t stream) {
  NI_CHECK_ARG(bgr && n_out && mask_out && H >= 1 && W >= 1, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(H) * W;
  int64_t blocks = (npix + 255) / 256;
  if (blocks > int64_t(kSMs) * 16) blocks = int64_t(kSMs) * 16;
  NI_COUNT_LAUNCH(), decode_png16_kernel<<<int(blocks), 256, 0, s>>>(bgr, npix, flip_z, n_out, mask_out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

// K9 -- gauge fix (pipeline.py:86-88, 229) and depth (geometry.py:180-184).
//
// median(z[valid]) per map by an exact MSB-first radix select over the
// order-preserving uint64 image of the float64 values (8 passes of 8 bits);
// numpy's even-count median is the mean of the two middle order statistics,
// (a + b) / 2, which both are selected in the same passes.
#include "ni_common.cuh"

namespace ni {

struct SelState {
  unsigned long long prefix[2];
  long long k[2];
  long long n;
};

__device__ __forceinline__ unsigned long long okey(double d) {
  unsigned long long u = __double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double from_okey(unsigned long long u) {
  u = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  return __longlong_as_double((long long)u);
}

__global__ void __launch_bounds__(256) select_hist_kernel(const double* __restrict__ z,
                                                          const uint8_t* __restrict__ valid,
                                                          int64_t per_map, int shift,
                                                          const SelState* __restrict__ st,
                                                          unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[2][256];
  const int m = blockIdx.y;
  for (int t = threadIdx.x; t < 512; t += blockDim.x) (&h[0][0])[t] = 0;
  __syncthreads();
  const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  const unsigned long long p0 = st[m].prefix[0] & hi_mask, p1 = st[m].prefix[1] & hi_mask;
  const int64_t base = int64_t(m) * per_map;
  // U independent loads in flight per thread (the pass is latency-bound
  // with one outstanding load per thread)
  constexpr int U = 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i0 < per_map;
       i0 += U * stride) {
    bool v[U];
    double zz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      v[u] = i < per_map && valid[base + i] != 0;
      zz[u] = i < per_map ? z[base + i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!v[u]) continue;
      const unsigned long long key = okey(zz[u]);
      const unsigned d = unsigned(key >> shift) & 255u;
      if ((key & hi_mask) == p0) atomicAdd(&h[0][d], 1u);
      if ((key & hi_mask) == p1) atomicAdd(&h[1][d], 1u);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 512; t += blockDim.x) {
    const unsigned v = (&h[0][0])[t];
    if (v) atomicAdd(hist + size_t(m) * 512 + t, v);
  }
}

__global__ void select_pick_kernel(unsigned int* __restrict__ hist, SelState* __restrict__ st,
                                   int shift, int B) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= B) return;
  SelState s = st[m];
  unsigned int* h = hist + size_t(m) * 512;
  if (shift == 56) {
    long long n = 0;
    for (int d = 0; d < 256; ++d) n += h[d];
    s.n = n;
    s.k[0] = n > 0 ? (n - 1) / 2 : 0;
    s.k[1] = n / 2;
    s.prefix[0] = s.prefix[1] = 0;
  }
  for (int sel = 0; sel < 2; ++sel) {
    long long acc = 0;
    int d = 0;
    for (; d < 255; ++d) {
      const long long c = h[sel * 256 + d];
      if (acc + c > s.k[sel]) break;
      acc += c;
    }
    s.k[sel] -= acc;
    s.prefix[sel] |= (unsigned long long)d << shift;
  }
  for (int t = 0; t < 512; ++t) h[t] = 0;
  st[m] = s;
}

__global__ void gauge_apply_kernel(double* __restrict__ z, const uint8_t* __restrict__ valid,
                                   int64_t per_map, const SelState* __restrict__ st, double target,
                                   double* __restrict__ depth, double* __restrict__ median_out) {
  const int m = blockIdx.y;
  const double a = from_okey(st[m].prefix[0]), b = from_okey(st[m].prefix[1]);
  const double med = (a + b) / 2.0;
  const double shift = target - med;
  if (median_out && blockIdx.x == 0 && threadIdx.x == 0) median_out[m] = med;
  const int64_t base = int64_t(m) * per_map;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per_map;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool v = valid[base + i] != 0;
    const double zz = v ? z[base + i] + shift : 0.0;
    z[base + i] = zz;
    if (depth) depth[base + i] = v ? exp(zz) : 0.0;
  }
}

}  // namespace ni

using namespace ni;

extern "C" int ni_gauge_workspace_size(int B, int H, int W, size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  Sizer z;
  z.take<SelState>(B);
  z.take<unsigned int>(size_t(B) * 512);
  z.take<double>(B);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_gauge(double* z, const uint8_t* valid, int B, int H, int W, double target,
                        double* depth_out, void* workspace, size_t workspace_bytes,
                        ni_stream_t stream) {
  NI_CHECK_ARG(z && valid && B >= 1, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  Carver c(workspace, workspace_bytes);
  SelState* st = c.take<SelState>(B);
  unsigned int* hist = c.take<unsigned int>(size_t(B) * 512);
  double* med = c.take<double>(B);
  if (!c.ok() || !workspace) {
    set_error("ni_gauge: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  const int64_t per_map = int64_t(H) * W;
  NI_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(SelState) * B, s));
  NI_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * size_t(B) * 512, s));
  int bx = int(std::min<int64_t>((per_map + 255) / 256, std::max<int64_t>(1, 4 * kSMs / B)));
  if (bx < 1) bx = 1;
  for (int shift = 56; shift >= 0; shift -= 8) {
    NI_COUNT_LAUNCH(), select_hist_kernel<<<dim3(bx, B), 256, 0, s>>>(z, valid, per_map, shift, st, hist);
    NI_COUNT_LAUNCH(), select_pick_kernel<<<div_up(B, 64), 64, 0, s>>>(hist, st, shift, B);
  }
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), gauge_apply_kernel<<<dim3(bx, B), 256, 0, s>>>(z, valid, per_map, st, target, depth_out, med);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

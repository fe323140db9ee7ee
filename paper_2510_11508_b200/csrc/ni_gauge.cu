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

// A warp per map: lane l owns bins 8 l .. 8 l + 7 of each histogram; the bin
// that holds the k-th element is found from a shuffle scan of the lane sums
// (the same bin and remainder as a serial walk over the 256 bins, which as a
// thread per map cost ~60 us per pass).
__global__ void __launch_bounds__(128) select_pick_kernel(unsigned int* __restrict__ hist,
                                                          SelState* __restrict__ st, int shift,
                                                          int B) {
  const int m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (m >= B) return;  // warp-uniform
  SelState s = st[m];
  unsigned int* h = hist + size_t(m) * 512;
  unsigned int bins[2][8];
#pragma unroll
  for (int sel = 0; sel < 2; ++sel)
#pragma unroll
    for (int j = 0; j < 8; ++j) bins[sel][j] = h[sel * 256 + lane * 8 + j];
  if (shift == 56) {
    long long n = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) n += bins[0][j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    s.n = n;
    s.k[0] = n > 0 ? (n - 1) / 2 : 0;
    s.k[1] = n / 2;
    s.prefix[0] = s.prefix[1] = 0;
  }
#pragma unroll
  for (int sel = 0; sel < 2; ++sel) {
    long long lsum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) lsum += bins[sel][j];
    long long incl = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long up = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += up;
    }
    const long long excl = incl - lsum;
    const unsigned found = __ballot_sync(0xffffffffu, incl > s.k[sel]);
    // the serial walk stops at bin 255 at the latest
    const int fl = found ? __ffs(found) - 1 : 31;
    long long acc = 0;
    int d = 0;
    if (lane == fl) {
      acc = excl;
      int j = 0;
      for (; j < 7; ++j) {
        const long long c = bins[sel][j];
        if (acc + c > s.k[sel]) break;
        acc += c;
      }
      d = lane * 8 + j;  // in the found lane the walk stops by j = 7: incl > k
    }
    acc = __shfl_sync(0xffffffffu, acc, fl);
    d = __shfl_sync(0xffffffffu, d, fl);
    s.k[sel] -= acc;
    s.prefix[sel] |= (unsigned long long)d << shift;
  }
#pragma unroll
  for (int sel = 0; sel < 2; ++sel)
#pragma unroll
    for (int j = 0; j < 8; ++j) h[sel * 256 + lane * 8 + j] = 0;
  if (lane == 0) st[m] = s;
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
    NI_COUNT_LAUNCH(), select_pick_kernel<<<div_up(B, 4), 128, 0, s>>>(hist, st, shift, B);
  }
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), gauge_apply_kernel<<<dim3(bx, B), 256, 0, s>>>(z, valid, per_map, st, target, depth_out, med);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

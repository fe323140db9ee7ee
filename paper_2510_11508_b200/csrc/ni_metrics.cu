// Depth-map evaluation on the GPU (metrics.py:44-113), batched over maps:
//
//  * ni_evaluate              evaluate(): median ratio alignment of the
//                             prediction (exact radix-select median, numpy's
//                             even-count convention), MADE and relative error
//                             over jointly valid pixels, per map
//  * ni_min_theoretical_made  min_theoretical_made(): every component gets its
//                             exactly L1-optimal scale -- the weighted median of
//                             its ratios gt/pred with weights pred, in stable
//                             ratio order with a sequential f64 cumsum like
//                             np.cumsum + searchsorted(side="left") -- then the
//                             pixel-count weighted mean error, per map
#include <cub/device/device_radix_sort.cuh>

#include "ni_common.cuh"

namespace ni {

// order-preserving uint64 image of a float64
__device__ __forceinline__ unsigned long long mkey(double d) {
  unsigned long long u = __double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double from_mkey(unsigned long long u) {
  u = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  return __longlong_as_double((long long)u);
}

// metrics.py:37-41: finite, positive, inside the mask
__global__ void ratio_kernel(const double* __restrict__ pred, const double* __restrict__ gt,
                             const uint8_t* __restrict__ mask, int64_t n,
                             double* __restrict__ ratio, uint8_t* __restrict__ ok) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double p = pred[i], g = gt[i];
    const bool v = isfinite(p) && isfinite(g) && p > 0.0 && g > 0.0 && (!mask || mask[i]);
    ok[i] = v;
    ratio[i] = v ? g / p : 0.0;
  }
}

// ---- median per map: MSB-first radix select of the two middle order
// statistics (8 passes of 8 bits over the order-preserving keys)
struct Sel {
  unsigned long long prefix[2];
  long long k[2];
  long long n;
};

__global__ void __launch_bounds__(256) sel_hist_kernel(const double* __restrict__ v,
                                                       const uint8_t* __restrict__ ok,
                                                       int64_t per_map, int shift,
                                                       const Sel* __restrict__ st,
                                                       unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[2][256];
  const int m = blockIdx.y;
  for (int t = threadIdx.x; t < 512; t += blockDim.x) (&h[0][0])[t] = 0;
  __syncthreads();
  const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  const unsigned long long p0 = st[m].prefix[0] & hi_mask, p1 = st[m].prefix[1] & hi_mask;
  const int64_t base = int64_t(m) * per_map;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per_map;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (!ok[base + i]) continue;
    const unsigned long long key = mkey(v[base + i]);
    const unsigned d = unsigned(key >> shift) & 255u;
    if ((key & hi_mask) == p0) atomicAdd(&h[0][d], 1u);
    if ((key & hi_mask) == p1) atomicAdd(&h[1][d], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 512; t += blockDim.x) {
    const unsigned c = (&h[0][0])[t];
    if (c) atomicAdd(hist + size_t(m) * 512 + t, c);
  }
}

__global__ void sel_pick_kernel(unsigned int* __restrict__ hist, Sel* __restrict__ st, int shift,
                                int B) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= B) return;
  Sel s = st[m];
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

// error sums per map at the median scale: one block per map, fixed order.
// out[4m .. 4m+3] = made, relative error, aligned scale, valid pixel count
__global__ void __launch_bounds__(256) made_kernel(const double* __restrict__ pred,
                                                   const double* __restrict__ gt,
                                                   const uint8_t* __restrict__ ok,
                                                   int64_t per_map, const Sel* __restrict__ st,
                                                   double* __restrict__ out) {
  __shared__ double red[32];
  const int m = blockIdx.x;
  const double scale = (from_mkey(st[m].prefix[0]) + from_mkey(st[m].prefix[1])) / 2.0;
  const int64_t base = int64_t(m) * per_map;
  double e = 0.0, r = 0.0;
  for (int64_t i = threadIdx.x; i < per_map; i += blockDim.x) {
    if (!ok[base + i]) continue;
    const double g = gt[base + i];
    const double err = fabs(scale * pred[base + i] - g);
    e += err;
    r += err / g;
  }
  e = block_sum(e, red);
  r = block_sum(r, red);
  if (threadIdx.x == 0) {
    const long long n = st[m].n;
    out[4 * m + 0] = n ? e / double(n) : 0.0;
    out[4 * m + 1] = n ? r / double(n) : 0.0;
    out[4 * m + 2] = scale;
    out[4 * m + 3] = double(n);
  }
}

// ---- min_theoretical_made
__global__ void comp_keys_kernel(const double* __restrict__ ratio, const uint8_t* __restrict__ ok,
                                 const int32_t* __restrict__ labels, int64_t n,
                                 unsigned long long* __restrict__ rkey,
                                 int32_t* __restrict__ lab, int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool v = ok[i] && labels[i] >= 0;
    rkey[i] = mkey(ratio[i]);
    lab[i] = v ? labels[i] : INT32_MAX;  // excluded pixels sort last
    idx[i] = int32_t(i);
  }
}

__global__ void run_start_kernel(const int32_t* __restrict__ lab_s, int64_t n,
                                 int32_t* __restrict__ flag) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x)
    flag[j] = (j == 0 || lab_s[j] != lab_s[j - 1]) ? 1 : 0;
}

__global__ void run_scatter_kernel(const int32_t* __restrict__ lab_s, const int32_t* __restrict__ flag,
                                   const int32_t* __restrict__ pos, int64_t n,
                                   int32_t* __restrict__ run_start, int32_t* __restrict__ run_lab,
                                   const int32_t* __restrict__ nruns) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    if (flag[j]) {
      run_start[pos[j]] = int32_t(j);
      run_lab[pos[j]] = lab_s[j];
    }
    if (j == 0) run_start[nruns[0]] = int32_t(n);
  }
}

// one thread per component run: its L1-optimal scale (metrics.py:68-84) and
// the sum of |s p - g| over its pixels
__global__ void comp_err_kernel(const int32_t* __restrict__ run_start,
                                const int32_t* __restrict__ run_lab,
                                const int32_t* __restrict__ nruns, const int32_t* __restrict__ idx_s,
                                const double* __restrict__ pred, const double* __restrict__ gt,
                                double* __restrict__ run_err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nruns[0]) return;
  const int s0 = run_start[c], s1 = run_start[c + 1];
  if (run_lab[c] == INT32_MAX) {
    run_err[c] = 0.0;
    return;
  }
  double total = 0.0;
  for (int j = s0; j < s1; ++j) total += pred[idx_s[j]];
  const double half = 0.5 * total;
  double cum = 0.0;
  int pick = s1 - 1;
  for (int j = s0; j < s1; ++j) {
    cum += pred[idx_s[j]];
    if (cum >= half) {  // np.searchsorted(cum, 0.5 * cum[-1], side="left")
      pick = j;
      break;
    }
  }
  const double s = gt[idx_s[pick]] / pred[idx_s[pick]];
  double e = 0.0;
  for (int j = s0; j < s1; ++j) {
    const int i = idx_s[j];
    e += fabs(s * pred[i] - gt[i]);
  }
  run_err[c] = e;
}

// per map: sum the errors and sizes of its components (label order)
__global__ void map_mtm_kernel(const int32_t* __restrict__ run_start,
                               const int32_t* __restrict__ run_lab,
                               const int32_t* __restrict__ nruns,
                               const double* __restrict__ run_err,
                               const int32_t* __restrict__ first, int B,
                               double* __restrict__ out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= B) return;
  const int lo = first[m], hi = first[m + 1];
  int a = 0, b = nruns[0];  // first run with label >= lo
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (run_lab[mid] < lo) a = mid + 1;
    else b = mid;
  }
  double err = 0.0;
  long long px = 0;
  for (int c = a; c < nruns[0] && run_lab[c] < hi; ++c) {
    err += run_err[c];
    px += run_start[c + 1] - run_start[c];
  }
  out[2 * m] = px ? err / double(px) : 0.0;
  out[2 * m + 1] = double(px);
}

__global__ void gather_kernel(const int32_t* __restrict__ v, const int32_t* __restrict__ idx,
                              int64_t n, int32_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x)
    out[j] = v[idx[j]];
}

static int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = int64_t(kSMs) * 16;
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace ni

using namespace ni;

extern "C" int ni_evaluate_workspace_size(int B, int H, int W, size_t* bytes) {
  NI_CHECK_ARG(bytes && B >= 1, "bad argument");
  const int64_t n = int64_t(B) * H * W;
  Sizer z;
  z.take<double>(n);
  z.take<uint8_t>(n);
  z.take<Sel>(B);
  z.take<unsigned int>(size_t(B) * 512);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_evaluate(const double* pred, const double* gt, const uint8_t* mask, int B, int H,
                           int W, double* out, void* workspace, size_t workspace_bytes,
                           ni_stream_t stream) {
  NI_CHECK_ARG(pred && gt && out && B >= 1, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t per_map = int64_t(H) * W, n = per_map * B;
  Carver c(workspace, workspace_bytes);
  double* ratio = c.take<double>(n);
  uint8_t* ok = c.take<uint8_t>(n);
  Sel* st = c.take<Sel>(B);
  unsigned int* hist = c.take<unsigned int>(size_t(B) * 512);
  if (!c.ok() || !workspace) {
    set_error("ni_evaluate: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  NI_COUNT_LAUNCH(), ratio_kernel<<<grid_for(n), 256, 0, s>>>(pred, gt, mask, n, ratio, ok);
  NI_LAUNCH_CHECK();
  NI_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(Sel) * B, s));
  NI_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * size_t(B) * 512, s));
  int bx = int(std::min<int64_t>((per_map + 255) / 256, std::max<int64_t>(1, 4 * kSMs / B)));
  if (bx < 1) bx = 1;
  for (int shift = 56; shift >= 0; shift -= 8) {
    NI_COUNT_LAUNCH(), sel_hist_kernel<<<dim3(bx, B), 256, 0, s>>>(ratio, ok, per_map, shift, st, hist);
    NI_COUNT_LAUNCH(), sel_pick_kernel<<<div_up(B, 64), 64, 0, s>>>(hist, st, shift, B);
  }
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), made_kernel<<<B, 256, 0, s>>>(pred, gt, ok, per_map, st, out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_min_theoretical_made_workspace_size(int B, int H, int W, size_t* bytes) {
  NI_CHECK_ARG(bytes && B >= 1, "bad argument");
  const int64_t n = int64_t(B) * H * W;
  Sizer z;
  z.take<double>(n);
  z.take<uint8_t>(n);
  z.take<unsigned long long>(n);
  z.take<unsigned long long>(n);
  for (int j = 0; j < 8; ++j) z.take<int32_t>(n + 2);
  z.take<double>(n + 1);
  z.take<int32_t>(B + 1);
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, int(n));
  cub::DeviceRadixSort::SortPairs(nullptr, b2, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, int(n));
  z.take<char>(b1 > b2 ? b1 : b2);
  z.take<char>(scan_ws_bytes(n + 1));
  *bytes = z.used;
  return NI_OK;
}

// labels: the partition's global labels (map m owns [map_first[m],
// map_first[m+1]) in HOST map_first[B+1]); out[2m] = the map's minimum
// theoretical MADE, out[2m+1] = its pixel count (0: no overlap).
extern "C" int ni_min_theoretical_made(const double* pred, const double* gt, const uint8_t* mask,
                                       const int32_t* labels, const int32_t* map_first, int B,
                                       int H, int W, double* out, void* workspace,
                                       size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(pred && gt && labels && map_first && out && B >= 1, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = int64_t(B) * H * W;
  NI_CHECK_ARG(n < (int64_t(1) << 31) - 2, "too many pixels");
  Carver c(workspace, workspace_bytes);
  double* ratio = c.take<double>(n);
  uint8_t* ok = c.take<uint8_t>(n);
  unsigned long long* rkey = c.take<unsigned long long>(n);
  unsigned long long* rkey_s = c.take<unsigned long long>(n);
  int32_t* lab = c.take<int32_t>(n + 2);
  int32_t* lab_a = c.take<int32_t>(n + 2);
  int32_t* lab_s = c.take<int32_t>(n + 2);
  int32_t* idx = c.take<int32_t>(n + 2);
  int32_t* idx_a = c.take<int32_t>(n + 2);
  int32_t* idx_s = c.take<int32_t>(n + 2);
  int32_t* flag = c.take<int32_t>(n + 2);
  int32_t* pos = c.take<int32_t>(n + 2);
  double* run_err = c.take<double>(n + 1);
  int32_t* first = c.take<int32_t>(B + 1);
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, int(n));
  cub::DeviceRadixSort::SortPairs(nullptr, b2, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, int(n));
  const size_t sb = b1 > b2 ? b1 : b2;
  void* sort_ws = c.take<char>(sb);
  void* scan_ws = c.take<char>(scan_ws_bytes(n + 1));
  if (!c.ok() || !workspace) {
    set_error("ni_min_theoretical_made: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  NI_CUDA_TRY(cudaMemcpyAsync(first, map_first, sizeof(int32_t) * (B + 1), cudaMemcpyHostToDevice, s));
  NI_COUNT_LAUNCH(), ratio_kernel<<<grid_for(n), 256, 0, s>>>(pred, gt, mask, n, ratio, ok);
  NI_COUNT_LAUNCH(), comp_keys_kernel<<<grid_for(n), 256, 0, s>>>(ratio, ok, labels, n, rkey, lab, idx);
  NI_LAUNCH_CHECK();
  // (label, ratio, pixel id) order: stable sort by ratio, then stable by label
  size_t t = sb;
  NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(sort_ws, t, rkey, rkey_s, idx, idx_a, int(n), 0, 64, s));
  // labels in the ratio order
  NI_COUNT_LAUNCH(), gather_kernel<<<grid_for(n), 256, 0, s>>>(lab, idx_a, n, lab_a);
  NI_LAUNCH_CHECK();
  t = sb;
  NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(sort_ws, t, lab_a, lab_s, idx_a, idx_s, int(n), 0, 32, s));
  NI_COUNT_LAUNCH(), run_start_kernel<<<grid_for(n), 256, 0, s>>>(lab_s, n, flag);
  NI_LAUNCH_CHECK();
  int32_t* nruns = pos + n + 1;
  NI_TRY(exclusive_scan_i32(flag, pos, n, nruns, scan_ws, s));
  int32_t* run_start = lab;  // reuse: [nruns + 1]
  int32_t* run_lab = idx;    // reuse: [nruns]
  NI_COUNT_LAUNCH(), run_scatter_kernel<<<grid_for(n), 256, 0, s>>>(lab_s, flag, pos, n, run_start, run_lab, nruns);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), comp_err_kernel<<<grid_for(n), 256, 0, s>>>(run_start, run_lab, nruns, idx_s, pred, gt, run_err);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), map_mtm_kernel<<<div_up(B, 64), 64, 0, s>>>(run_start, run_lab, nruns, run_err, first, B, out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

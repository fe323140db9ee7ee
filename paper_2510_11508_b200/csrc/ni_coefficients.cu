// K2 -- per-edge continuity coefficients (continuity.py:210-289), float64.
//
// One thread per pixel a evaluates its KF forward edges; coefficients are
// stored as KF planes (omega_a[k*npix + a]) so every later pass reads them
// coalesced.  gamma (continuity.py:270-274) depends only on the pixel, so it
// is stored once per pixel instead of twice per edge.
#include "ni_common.cuh"

namespace ni {

constexpr double kEpsDen = 1e-8;   // continuity.py:34
constexpr double kEpsLog = 1e-12;  // continuity.py:35

// A CTA covers a 32-column x CROWS-row tile of the stacked B*H rows: a
// thread owns one column and walks the rows, so the ray components that
// depend on the column only ((u - cx) / fx at u, u +- 1 and at the midpoints)
// are divided once per column and those that depend on the row only once per
// row (in shared memory).  Same operands and operation order as a per-edge
// evaluation, so every value is bit-identical to the reference's.
constexpr int CCOLS = 32, CTHR_Y = 8, CROWS = 32;

struct ColRays {
  int m = -1;
  double t0, tp, tm, hp, hm;  // (u - cx)/fx at u, u+1, u-1 and the midpoints u+-1/2
};

template <int CONN, int MODEL>
__global__ void __launch_bounds__(CCOLS * CTHR_Y) coefficients_kernel(
    const double* __restrict__ n, const uint8_t* __restrict__ valid,
    const double* __restrict__ intr, int H, int W, int64_t npix, double* __restrict__ omega_a,
    double* __restrict__ omega_b, double* __restrict__ gamma, uint8_t* __restrict__ eflags,
    ni_stats* __restrict__ st, long long* __restrict__ map_counts) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  __shared__ double s_t0[CROWS], s_tp[CROWS], s_hp[CROWS];  // (v - cy)/fy at v, v+1, v+1/2
  const int rows = int(npix / W);
  const int row0 = blockIdx.y * CROWS;
  const int u = blockIdx.x * CCOLS + threadIdx.x;
  const int tid = threadIdx.y * CCOLS + threadIdx.x;
  if (tid < CROWS && row0 + tid < rows) {
    const int r = row0 + tid;
    const int m = r / H;
    const double fy = intr[4 * m + 1], cy = intr[4 * m + 3];
    const double va = double(r - m * H);
    s_t0[tid] = (va - cy) / fy;
    s_tp[tid] = (va + 1.0 - cy) / fy;
    s_hp[tid] = (0.5 * (va + (va + 1.0)) - cy) / fy;
  }
  // per-map edge / degenerate-edge counts of this tile's rows (maps m0 ..):
  // a warp (one row) reduces its lanes' counts, lane 0 adds them to a 32-bit
  // shared counter (<= 4096 per tile), one global atomic per map and counter.
  // (Per-thread 64-bit shared atomics were a CAS loop under contention that
  // cost more than the coefficients themselves.)
  __shared__ unsigned s_cnt[CROWS][2];
  const int m0 = row0 / H;
  if (tid < CROWS) s_cnt[tid][0] = s_cnt[tid][1] = 0u;
  __syncthreads();
  long long ndegen = 0;
  ColRays cr;
  const bool in_cols = u < W;
  for (int ry = threadIdx.y; ry < CROWS; ry += CTHR_Y) {
    const int row = row0 + ry;
    if (row >= rows) break;  // uniform over the warp (one row)
    const int m = row / H;
    if (!in_cols) {
      if (map_counts) {  // the warp's reduction needs every lane
        __reduce_add_sync(0xffffffffu, 0u);
        __reduce_add_sync(0xffffffffu, 0u);
      }
      continue;
    }
    const int vloc = row - m * H;
    const int64_t i = int64_t(row) * W + u;
    const double fx = intr[4 * m + 0], fy = intr[4 * m + 1];
    if (cr.m != m) {
      const double cx = intr[4 * m + 2];
      const double ua = double(u);
      cr.m = m;
      cr.t0 = (ua - cx) / fx;
      cr.tp = (ua + 1.0 - cx) / fx;
      cr.tm = (ua + -1.0 - cx) / fx;
      cr.hp = (0.5 * (ua + (ua + 1.0)) - cx) / fx;
      cr.hm = (0.5 * (ua + (ua + -1.0)) - cx) / fx;
    }
    uint8_t flags = 0;
    double g = 0.0;
    double om_a[KF], om_b[KF];
#pragma unroll
    for (int k = 0; k < KF; ++k) om_a[k] = om_b[k] = 0.0;
    if (valid[i]) {
      const double a0 = n[i], a1 = n[npix + i], a2 = n[2 * npix + i];
      const double ta0 = cr.t0, ta1 = s_t0[ry];
      // gamma = mean_focal * |n . tau / ||tau|| |   (continuity.py:270-274)
      const double tn = sqrt(ta0 * ta0 + ta1 * ta1 + 1.0);
      g = 0.5 * (fx + fy) * fabs(a0 * (ta0 / tn) + a1 * (ta1 / tn) + a2 * (1.0 / tn));
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
        if (!fwd_inside(u, vloc, du, dv, W, H)) continue;
        const int64_t j = i + int64_t(dv) * W + du;
        if (!valid[j]) continue;
        flags |= uint8_t(1u << k);
        const double b0 = n[j], b1 = n[npix + j], b2 = n[2 * npix + j];
        bool ok;
        if (MODEL == 0) {  // milano, continuity.py:232-247
          // (ub - cx) / fx, (vb - cy) / fy, (0.5 (ua + ub) - cx) / fx, (0.5 (va + vb) - cy) / fy
          const double tb0 = du > 0 ? cr.tp : (du < 0 ? cr.tm : ta0);
          const double tb1 = dv > 0 ? s_tp[ry] : ta1;
          const double tm0 = du > 0 ? cr.hp : (du < 0 ? cr.hm : ta0);
          const double tm1 = dv > 0 ? s_hp[ry] : ta1;
          const double pa = a0 * ta0 + a1 * ta1 + a2;
          const double pb = b0 * tb0 + b1 * tb1 + b2;
          const double ma = a0 * tm0 + a1 * tm1 + a2;
          const double mb = b0 * tm0 + b1 * tm1 + b2;
          const double small = fmin(fmin(fabs(pa), fabs(pb)), fmin(fabs(ma), fabs(mb)));
          const double arg = (ma * pb) / (pa * mb);
          ok = small >= kEpsDen && arg > kEpsLog;
          if (ok) {
            om_a[k] = log(arg);
            om_b[k] = -om_a[k];
          }
        } else {  // bini, continuity.py:248-268 (axis-aligned edges only)
          const double cx = intr[4 * m + 2], cy = intr[4 * m + 3];
          const double ua = double(u), va = double(vloc);
          const double ub = ua + du, vb = va + dv;
          const bool horiz = dv == 0;
          const double f = horiz ? fx : fy;
          const double num_a = horiz ? du * a0 : dv * a1;
          const double num_b = horiz ? -du * b0 : -dv * b1;
          const double den_a = a0 * (ua - cx) + a1 * (va - cy) + a2 * f;
          const double den_b = b0 * (ub - cx) + b1 * (vb - cy) + b2 * f;
          ok = fabs(den_a) >= kEpsDen && fabs(den_b) >= kEpsDen;
          if (ok) {
            om_a[k] = num_a / den_a;
            om_b[k] = num_b / den_b;
          }
        }
        if (ok) flags |= uint8_t(1u << (4 + k));
        else ++ndegen;
      }
    }
    gamma[i] = g;
    eflags[i] = flags;
    if (map_counts) {
      const unsigned nex = __popc(flags & 0xfu), nok = __popc(flags >> 4);
      const unsigned wex = __reduce_add_sync(0xffffffffu, nex);
      const unsigned wdg = __reduce_add_sync(0xffffffffu, nex - nok);
      if (threadIdx.x == 0) {
        if (wex) atomicAdd(&s_cnt[m - m0][0], wex);
        if (wdg) atomicAdd(&s_cnt[m - m0][1], wdg);
      }
    }
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      omega_a[k * npix + i] = om_a[k];
      if (MODEL == 1) omega_b[k * npix + i] = om_b[k];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ndegen += __shfl_xor_sync(0xffffffffu, ndegen, o);
  if ((threadIdx.x & 31) == 0 && ndegen)
    atomicAdd((unsigned long long*)&st->degenerate_edges, (unsigned long long)ndegen);
  if (map_counts) {
    __syncthreads();
    if (tid < CROWS) {
      const int m = m0 + tid;
      if (s_cnt[tid][0])
        atomicAdd((unsigned long long*)&map_counts[2 * m], (unsigned long long)s_cnt[tid][0]);
      if (s_cnt[tid][1])
        atomicAdd((unsigned long long*)&map_counts[2 * m + 1], (unsigned long long)s_cnt[tid][1]);
    }
  }
}

}  // namespace ni

using namespace ni;

extern "C" int ni_coefficients(const double* n, const uint8_t* valid, const double* intrinsics, int B,
                               int H, int W, int connectivity, int model, double* omega_a,
                               double* omega_b, double* gamma, uint8_t* eflags, ni_stats* stats,
                               long long* map_counts, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(model == 0 || model == 1, "model must be 0 (milano) or 1 (bini)");
  NI_CHECK_ARG(!(model == 1 && connectivity == 8),
               "the pinhole finite-difference model defines no diagonal coefficient; use "
               "connectivity=4 with model='bini'");
  NI_CHECK_ARG(n && valid && intrinsics && omega_a && gamma && eflags && stats, "null pointer");
  NI_CHECK_ARG(model == 0 || omega_b, "bini needs omega_b");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  NI_CUDA_TRY(cudaMemsetAsync(&stats->degenerate_edges, 0, sizeof(long long), s));
  if (map_counts) NI_CUDA_TRY(cudaMemsetAsync(map_counts, 0, sizeof(long long) * 2 * B, s));
  const dim3 blocks(unsigned(div_up(W, CCOLS)), unsigned(div_up(B * H, CROWS)));
  const dim3 threads(CCOLS, CTHR_Y);
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), coefficients_kernel<8, 0><<<blocks, threads, 0, s>>>(n, valid, intrinsics, H, W, npix, omega_a,
                                                     omega_b, gamma, eflags, stats, map_counts);
  else if (model == 0)
    NI_COUNT_LAUNCH(), coefficients_kernel<4, 0><<<blocks, threads, 0, s>>>(n, valid, intrinsics, H, W, npix, omega_a,
                                                     omega_b, gamma, eflags, stats, map_counts);
  else
    NI_COUNT_LAUNCH(), coefficients_kernel<4, 1><<<blocks, threads, 0, s>>>(n, valid, intrinsics, H, W, npix, omega_a,
                                                     omega_b, gamma, eflags, stats, map_counts);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

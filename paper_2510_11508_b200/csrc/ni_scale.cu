// K4-K8: the relative-scale loop over the quotient graph.
//
//  * ni_inter_edges      graph.py:186-196   ordered compaction of inter edges
//  * ni_quotient_build   solver.py:153-180  static structure of the pair system
//                                           (pair runs, component incidence,
//                                           Laplacian sparsity) per partition
//  * ni_scale_step       solver.py:253-303  weights (K4), segmented pair sums
//                                           (K5), small CG (K6), residuals +
//                                           energy, z += s[label] (K7,
//                                           pipeline.py:181-182)
//  * ni_merge            graph.py:207-250 + pipeline.py:187-203  (K8)
//
// Every floating-point sum runs in a fixed order (runs sorted by edge index,
// block partials summed in block order), so reruns are bit-identical.
#include <cooperative_groups.h>

#include <cub/device/device_radix_sort.cuh>

#include "ni_common.cuh"

namespace cg = cooperative_groups;

namespace ni {

// ------------------------------------------------------------ inter edges

template <int CONN>
__global__ void inter_flags_kernel(const int32_t* __restrict__ labels,
                                   const uint8_t* __restrict__ eflags, int W, int64_t npix,
                                   int32_t* __restrict__ flag) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t ef = eflags[i];
    const int32_t la = labels[i];
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      int f = 0;
      if ((ef >> k) & 1) {
        const int64_t j = i + int64_t(fwd_dv(CONN, k)) * W + fwd_du(CONN, k);
        f = labels[j] != la;
      }
      flag[i * KF + k] = f;
    }
  }
}

__global__ void compact_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                               int64_t n, int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    if (flag[e]) out[pos[e]] = int32_t(e);
}

// ------------------------------------------------------- quotient layout

struct Quot {
  int K, C;
  int32_t* ea;        // [K] pixel a
  int32_t* eb;        // [K] pixel b
  int32_t* ek;        // [K] direction
  int32_t* pa;        // [K] component of a (local, 0..C-1)
  int32_t* pb;        // [K] component of b
  int32_t* order;     // [K] edges sorted by (min, max) component pair
  int32_t* pstart;    // [K+1] pair runs in `order`; first U+1 used
  int32_t* pp;        // [K] pair endpoints (p < q)
  int32_t* pq;        // [K]
  int32_t* cstart;    // [C+1] incidence runs
  int32_t* cent;      // [2K] 2*e + side (0: component is pa, 1: pb)
  int32_t* lstart;    // [C+1] Laplacian rows
  int32_t* lcol;      // [2K] column
  int32_t* lpair;     // [2K] pair index
  int32_t* nU;        // [1]
  // scratch used while building
  long long* k64a;
  long long* k64b;
  int32_t* v32a;
  int32_t* v32b;
  int32_t* flag;
  int32_t* hist;
  void* sort_ws;
  size_t sort_bytes;
  void* scan_ws;
};

static void carve_quot(Carver& c, Quot& q, int K, int C) {
  const int64_t K2 = 2 * int64_t(K) + 1;
  q.K = K;
  q.C = C;
  q.ea = c.take<int32_t>(K + 1);
  q.eb = c.take<int32_t>(K + 1);
  q.ek = c.take<int32_t>(K + 1);
  q.pa = c.take<int32_t>(K + 1);
  q.pb = c.take<int32_t>(K + 1);
  q.order = c.take<int32_t>(K + 1);
  q.pstart = c.take<int32_t>(K + 2);
  q.pp = c.take<int32_t>(K + 1);
  q.pq = c.take<int32_t>(K + 1);
  q.cstart = c.take<int32_t>(C + 2);
  q.cent = c.take<int32_t>(K2);
  q.lstart = c.take<int32_t>(C + 2);
  q.lcol = c.take<int32_t>(K2);
  q.lpair = c.take<int32_t>(K2);
  q.nU = c.take<int32_t>(1);
  q.k64a = c.take<long long>(K2);
  q.k64b = c.take<long long>(K2);
  q.v32a = c.take<int32_t>(K2);
  q.v32b = c.take<int32_t>(K2);
  q.flag = c.take<int32_t>(K2);
  q.hist = c.take<int32_t>(C + 2);
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b1, (const long long*)nullptr, (long long*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)K2);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)K2);
  q.sort_bytes = b1 > b2 ? b1 : b2;
  q.sort_ws = c.take<char>(q.sort_bytes);
  q.scan_ws = c.take<char>(scan_ws_bytes(K2 > C + 2 ? K2 : C + 2));
}

template <int CONN>
__global__ void quot_edges_kernel(const int32_t* __restrict__ keys, int K,
                                  const int32_t* __restrict__ labels, int label_base, int W, int C,
                                  Quot q) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K; e += gridDim.x * blockDim.x) {
    const int32_t key = keys[e];
    const int32_t a = key / KF, k = key % KF;
    const int32_t b = a + fwd_dv(CONN, k) * W + fwd_du(CONN, k);
    const int32_t la = labels[a] - label_base, lb = labels[b] - label_base;
    q.ea[e] = a;
    q.eb[e] = b;
    q.ek[e] = k;
    q.pa[e] = la;
    q.pb[e] = lb;
    const int32_t lo = la < lb ? la : lb, hi = la < lb ? lb : la;
    q.k64a[e] = (long long)lo * C + hi;
    q.v32a[e] = e;
    // incidence entries
    q.v32b[2 * e] = 2 * e;
    q.v32b[2 * e + 1] = 2 * e + 1;
    q.flag[2 * e] = la;
    q.flag[2 * e + 1] = lb;
  }
}

__global__ void pair_runs_kernel(const long long* __restrict__ sk, int K, int C,
                                 const int32_t* __restrict__ runpos, Quot q) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x) {
    if (j == 0 || sk[j] != sk[j - 1]) {
      const int u = runpos[j];
      q.pstart[u] = j;
      q.pp[u] = int32_t(sk[j] / C);
      q.pq[u] = int32_t(sk[j] % C);
    }
  }
}

__global__ void run_flags_kernel(const long long* __restrict__ sk, int n, int32_t* __restrict__ f) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    f[j] = (j == 0 || sk[j] != sk[j - 1]) ? 1 : 0;
}

__global__ void set_tail_kernel(int32_t* __restrict__ arr, const int32_t* __restrict__ idx, int val) {
  arr[idx[0]] = val;
}

__global__ void hist_kernel(const int32_t* __restrict__ keys, int n, int32_t* __restrict__ hist) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    atomicAdd(hist + keys[j], 1);
}

__global__ void lap_entries_kernel(Quot q, const int32_t* __restrict__ nU_dev) {
  const int U = nU_dev[0];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    const int32_t p = q.pp[u], r = q.pq[u];
    q.k64a[2 * u] = (long long)p * q.C + r;
    q.k64a[2 * u + 1] = (long long)r * q.C + p;
    q.v32a[2 * u] = u;
    q.v32a[2 * u + 1] = u;
    q.flag[2 * u] = p;
    q.flag[2 * u + 1] = r;
  }
}

__global__ void lap_cols_kernel(Quot q, const long long* __restrict__ sk, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    q.lcol[j] = int32_t(sk[j] % q.C);
}

static int blocks_for(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  if (b < 1) b = 1;
  if (b > int64_t(kSMs) * 8) b = int64_t(kSMs) * 8;
  return int(b);
}

static int end_bits_for(int64_t maxval) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) <= maxval) ++b;
  return b;
}

// ------------------------------------------------------------ scale step

struct StepWs {
  double *wa, *wb, *ba, *bb, *S, *diag, *rhs, *s, *r, *p0, *p1, *q, *part;
  double* epart;
  int32_t *anyflag, *parent, *pflag, *prank, *ptotal, *pkey, *pkey_s, *pval, *pval_s, *okflag;
  void* sort_ws;
  size_t sort_bytes;
  void* scan_ws;
};

constexpr int kCgThreads = 512;
constexpr int kResBlocks = 296;

static void carve_step(Carver& c, StepWs& w, int K, int C) {
  w.wa = c.take<double>(K + 1);
  w.wb = c.take<double>(K + 1);
  w.ba = c.take<double>(K + 1);
  w.bb = c.take<double>(K + 1);
  w.S = c.take<double>(K + 1);
  w.diag = c.take<double>(C + 1);
  w.rhs = c.take<double>(C + 1);
  w.s = c.take<double>(C + 1);
  w.r = c.take<double>(C + 1);
  w.p0 = c.take<double>(C + 1);
  w.p1 = c.take<double>(C + 1);
  w.q = c.take<double>(C + 1);
  w.part = c.take<double>(4 * kSMs + 8);
  w.epart = c.take<double>(kResBlocks + 1);
  w.anyflag = c.take<int32_t>(1);
  w.okflag = c.take<int32_t>(1);
  w.parent = c.take<int32_t>(C + 1);
  w.pflag = c.take<int32_t>(C + 1);
  w.prank = c.take<int32_t>(C + 1);
  w.ptotal = c.take<int32_t>(1);
  w.pkey = c.take<int32_t>(C + 1);
  w.pkey_s = c.take<int32_t>(C + 1);
  w.pval = c.take<int32_t>(C + 1);
  w.pval_s = c.take<int32_t>(C + 1);
  w.sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, w.sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, C + 1);
  w.sort_ws = c.take<char>(w.sort_bytes);
  w.scan_ws = c.take<char>(scan_ws_bytes(C + 2));
}

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// K4: weights and row right-hand sides (solver.py:253-278, 170-180)
template <int CONN, int MODEL>
__global__ void weights_kernel(Quot q, const double* __restrict__ z,
                               const double* __restrict__ omega_a,
                               const double* __restrict__ omega_b,
                               const double* __restrict__ gamma,
                               const uint8_t* __restrict__ eflags, int H, int W, int64_t npix,
                               int uniform, int mode, double kk, double lt, double ut,
                               double hi, StepWs w) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < q.K; e += gridDim.x * blockDim.x) {
    const int32_t a = q.ea[e], b = q.eb[e], k = q.ek[e];
    const uint8_t efa = eflags[a];
    const bool valid = (efa >> (4 + k)) & 1;
    const double za = z[a], zb = z[b];
    const double oa = omega_a[k * npix + a];
    const double ob = MODEL == 0 ? -oa : omega_b[k * npix + a];
    double wa = 0.0, wb = 0.0;
    if (valid) {
      if (uniform) {
        wa = wb = 1.0;
      } else {
        const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
        // opposite of b through a: a - off (continuity.py:196-207, 276)
        const int ua = a % W, va = (a / W) % H;
        const int uo = ua - du, vo = va - dv;
        bool has_a = false;
        double zoa = 0.0;
        if (uo >= 0 && uo < W && vo >= 0) {
          const int32_t o = a - dv * W - du;
          if ((eflags[o] >> k) & 1) {  // edge o -> a exists: o valid, same map
            has_a = true;
            zoa = z[o];
          }
        }
        const bool has_b = (eflags[b] >> k) & 1;  // b + off exists
        const double zob = has_b ? z[b + dv * W + du] : 0.0;
        const double ga = gamma[a], gb = gamma[b];
        const double g2a = ga * ga, g2b = gb * gb;
        double bil_a = 0.5, bil_b = 0.5;
        if (has_a) {
          const double dp = zoa - za, dq = zb - za;
          bil_a = sigmoid(kk * (g2a * (dp * dp - dq * dq)));
        }
        if (has_b) {
          const double dp = zob - zb, dq = za - zb;
          bil_b = sigmoid(kk * (g2b * (dp * dp - dq * dq)));
        }
        wa = g2a * bil_a;
        wb = g2b * bil_b;
        // outlier weights on chi (continuity.py:140-158)
        const double chia = za - zb - oa, chib = zb - za - ob;
        if (mode == 1) {
          const double ca = fabs(chia) > 1e-300 ? fabs(chia) : 1e-300;
          const double cb = fabs(chib) > 1e-300 ? fabs(chib) : 1e-300;
          const double sc = 4.0 / (lt - ut);
          wa *= sigmoid(sc * (2.0 * log10(ca) - (lt + ut)));
          wb *= sigmoid(sc * (2.0 * log10(cb) - (lt + ut)));
        } else if (mode == 2) {
          if (fabs(chia) >= hi) wa = 0.0;
          if (fabs(chib) >= hi) wb = 0.0;
        }
      }
    }
    w.wa[e] = wa;
    w.wb[e] = wb;
    w.ba[e] = oa - (za - zb);
    w.bb[e] = ob - (zb - za);
  }
}

// K5a: conductance per component pair, summed over its run in edge order.
// One warp per pair: lane-strided partial sums then a fixed xor tree.
__global__ void pair_sum_kernel(Quot q, StepWs w, const int32_t* __restrict__ nU_dev) {
  const int U = nU_dev[0];
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += warps) {
    double s = 0.0;
    for (int j = q.pstart[u] + lane; j < q.pstart[u + 1]; j += 32) {
      const int e = q.order[j];
      s += w.wa[e] + w.wb[e];
    }
    s = warp_sum(s);
    if (lane == 0) w.S[u] = s;
  }
}

// K5b: diagonal and A^T W b per component, summed over its incident edges in
// edge order (solver.py:108-111).  One warp per component.
__global__ void comp_sum_kernel(Quot q, StepWs w) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < q.C; c += warps) {
    double d = 0.0, r = 0.0;
    for (int j = q.cstart[c] + lane; j < q.cstart[c + 1]; j += 32) {
      const int ent = q.cent[j];
      const int e = ent >> 1;
      const double wa = w.wa[e], wb = w.wb[e];
      const double t = wa * w.ba[e] - wb * w.bb[e];
      d += wa + wb;
      r += (ent & 1) ? -t : t;
    }
    d = warp_sum(d);
    r = warp_sum(r);
    if (lane == 0) {
      w.diag[c] = d;
      w.rhs[c] = r;
      if (r != 0.0) atomicOr(w.anyflag, 1);
    }
  }
}

// roundoff null-space removal: parts = components connected by S > 0
__global__ void part_init_kernel(StepWs w, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    w.parent[c] = c;
}

__global__ void part_union_kernel(Quot q, StepWs w, const int32_t* __restrict__ nU_dev) {
  const int U = nU_dev[0];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x)
    if (w.S[u] > 0.0) uf_union(w.parent, q.pp[u], q.pq[u]);
}

__global__ void part_flatten_kernel(StepWs w, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int r = uf_find(w.parent, c);
    w.pkey[c] = r;
    w.pval[c] = c;
  }
}

// one warp per part segment (components sorted by part root, ascending)
__global__ void part_mean_kernel(StepWs w, int C) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < C; j += warps) {
    if (j > 0 && w.pkey_s[j] == w.pkey_s[j - 1]) continue;
    const int key = w.pkey_s[j];
    int e = j;
    double s = 0.0;
    // walk the segment 32 entries at a time
    while (true) {
      const int t = e + lane;
      const bool in = t < C && w.pkey_s[t] == key;
      if (in) s += w.rhs[w.pval_s[t]];
      const unsigned b = __ballot_sync(0xffffffffu, in);
      e += __popc(b);
      if (b != 0xffffffffu) break;
    }
    s = warp_sum(s);
    const double mean = s / double(e - j);
    for (int t = j + lane; t < e; t += 32) w.r[w.pval_s[t]] = mean;  // stash mean per comp
  }
}

__global__ void part_sub_kernel(StepWs w, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    w.rhs[c] = w.rhs[c] - w.r[c];
}

// K6: scipy-equivalent CG on the component Laplacian (solver.py:97-122).
// Cooperative kernel; every block redundantly sums the per-block partials in
// block order, so all blocks agree bit for bit on every scalar.
__device__ __forceinline__ double grid_sum(cg::grid_group& grid, double v, double* part, int slot,
                                           double* red) {
  v = block_sum(v, red);
  if (threadIdx.x == 0) part[slot * gridDim.x + blockIdx.x] = v;
  grid.sync();
  double t = 0.0;
  for (int b = 0; b < int(gridDim.x); ++b) t += __ldcg(part + slot * gridDim.x + b);
  return t;
}

__global__ void __launch_bounds__(kCgThreads) scale_cg_kernel(Quot q, StepWs w, double rtol,
                                                              int maxiter) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  const int C = q.C;
  const int tid0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  double rr = 0.0;
  for (int c = tid0; c < C; c += stride) {
    const double b = w.rhs[c];
    w.s[c] = 0.0;
    w.r[c] = b;
    w.p0[c] = 0.0;
    rr += b * b;
  }
  rr = grid_sum(grid, rr, w.part, 0, red);
  const double bnrm = sqrt(rr);
  if (bnrm == 0.0) {
    if (tid0 == 0) w.okflag[0] = 1;
    return;
  }
  const double atol = rtol * bnrm;
  double rho_prev = 0.0;
  double* pold = w.p0;
  double* pnew = w.p1;
  int ok = 0;
  for (int it = 0; it < maxiter; ++it) {
    if (sqrt(rr) < atol) {
      ok = 1;
      break;
    }
    const double rho = rr;
    const double beta = it == 0 ? 0.0 : rho / rho_prev;
    double pq = 0.0;
    for (int c = tid0; c < C; c += stride) {
      const double pc = w.r[c] + beta * pold[c];
      double acc = w.diag[c] * pc;
      for (int j = q.lstart[c]; j < q.lstart[c + 1]; ++j) {
        const int nb = q.lcol[j];
        acc -= w.S[q.lpair[j]] * (w.r[nb] + beta * pold[nb]);
      }
      pnew[c] = pc;
      w.q[c] = acc;
      pq += pc * acc;
    }
    pq = grid_sum(grid, pq, w.part, 1, red);
    const double alpha = rho / pq;
    double rn = 0.0;
    for (int c = tid0; c < C; c += stride) {
      w.s[c] += alpha * pnew[c];
      const double r2 = w.r[c] - alpha * w.q[c];
      w.r[c] = r2;
      rn += r2 * r2;
    }
    rr = grid_sum(grid, rn, w.part, 2 + (it & 1), red);
    rho_prev = rho;
    double* t = pold;
    pold = pnew;
    pnew = t;
  }
  if (tid0 == 0) w.okflag[0] = ok;
}

// K7a: residual rows and the energy (solver.py:301-302)
__global__ void __launch_bounds__(256) residual_kernel(Quot q, StepWs w, double* __restrict__ scales,
                                                       double* __restrict__ residual,
                                                       double* __restrict__ weights) {
  __shared__ double red[32];
  double en = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < q.K; e += gridDim.x * blockDim.x) {
    const double sa = w.s[q.pa[e]], sb = w.s[q.pb[e]];
    const double ra = sa - sb - w.ba[e];
    const double rb = sb - sa - w.bb[e];
    residual[2 * e] = ra;
    residual[2 * e + 1] = rb;
    weights[2 * e] = w.wa[e];
    weights[2 * e + 1] = w.wb[e];
    en += ra * (w.wa[e] * ra) + rb * (w.wb[e] * rb);
  }
  en = block_sum(en, red);
  if (threadIdx.x == 0) w.epart[blockIdx.x] = en;
}

__global__ void energy_final_kernel(StepWs w, int nblocks, double* __restrict__ scales_out, int C,
                                    double* __restrict__ energy_out, int32_t* __restrict__ ok_out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double e = 0.0;
    for (int b = 0; b < nblocks; ++b) e += w.epart[b];
    energy_out[0] = e;
    ok_out[0] = w.okflag[0];
  }
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    scales_out[c] = w.s[c];
}

// K7b: z[valid] += s[label] on the map's pixel range (pipeline.py:181-182)
__global__ void apply_kernel(double* __restrict__ z, const int32_t* __restrict__ labels,
                             const double* __restrict__ s, int label_base, int64_t p0, int64_t p1) {
  for (int64_t i = p0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < p1;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t l = labels[i];
    if (l >= 0) z[i] += s[l - label_base];
  }
}

__global__ void set_int_kernel(int32_t* __restrict__ a, int v) { a[0] = v; }

__global__ void zero_kernel(double* __restrict__ a, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) a[j] = 0.0;
}

// ----------------------------------------------------------------- merge

struct MergeWs {
  int32_t *sel, *parent, *flag, *rank, *total;
  double* epart;
  void* scan_ws;
};

static void carve_merge(Carver& c, MergeWs& m, int K, int C) {
  m.sel = c.take<int32_t>(C + 1);
  m.parent = c.take<int32_t>(C + 1);
  m.flag = c.take<int32_t>(C + 1);
  m.rank = c.take<int32_t>(C + 1);
  m.total = c.take<int32_t>(1);
  m.epart = c.take<double>(kResBlocks + 1);
  m.scan_ws = c.take<char>(scan_ws_bytes(C + 2));
}

// argmin over incident inter edges of (|residual_a|, edge index)
// (graph.py:230-239); one warp per component, lexicographic warp argmin.
__global__ void merge_select_kernel(Quot q, const double* __restrict__ residual, MergeWs m) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < q.C; c += warps) {
    int best_e = -1;
    double best = 0.0;
    for (int j = q.cstart[c] + lane; j < q.cstart[c + 1]; j += 32) {
      const int e = q.cent[j] >> 1;
      const double r = fabs(residual[2 * e]);
      if (best_e < 0 || r < best || (r == best && e < best_e)) {
        best = r;
        best_e = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oe = __shfl_xor_sync(0xffffffffu, best_e, o);
      if (oe >= 0 && (best_e < 0 || ob < best || (ob == best && oe < best_e))) {
        best = ob;
        best_e = oe;
      }
    }
    if (lane == 0) {
      m.sel[c] = best_e;
      m.parent[c] = c;
    }
  }
}

__global__ void merge_union_kernel(Quot q, MergeWs m) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < q.C; c += gridDim.x * blockDim.x) {
    const int e = m.sel[c];
    if (e >= 0) uf_union(m.parent, q.pa[e], q.pb[e]);
  }
}

__global__ void merge_flatten_kernel(MergeWs m, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int r = uf_find(m.parent, c);
    m.parent[c] = r;
    m.flag[c] = r == c;
  }
}

__global__ void merge_relabel_kernel(int32_t* __restrict__ labels, const MergeWs m, int label_base,
                                     int64_t p0, int64_t p1) {
  for (int64_t i = p0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < p1;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t l = labels[i];
    if (l >= 0) labels[i] = label_base + m.rank[m.parent[l - label_base]];
  }
}

// energy restricted to edges that stay inter-component (pipeline.py:196-203)
__global__ void __launch_bounds__(256) merge_energy_kernel(Quot q, const MergeWs m,
                                                           const double* __restrict__ residual,
                                                           const double* __restrict__ weights) {
  __shared__ double red[32];
  double en = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < q.K; e += gridDim.x * blockDim.x) {
    if (m.parent[q.pa[e]] != m.parent[q.pb[e]]) {
      const double ra = residual[2 * e], rb = residual[2 * e + 1];
      en += ra * (weights[2 * e] * ra) + rb * (weights[2 * e + 1] * rb);
    }
  }
  en = block_sum(en, red);
  if (threadIdx.x == 0) m.epart[blockIdx.x] = en;
}

__global__ void merge_final_kernel(const MergeWs m, int nblocks, double* __restrict__ energy_out,
                                   int32_t* __restrict__ count_out) {
  double e = 0.0;
  for (int b = 0; b < nblocks; ++b) e += m.epart[b];
  energy_out[0] = e;
  count_out[0] = m.total[0];
}

}  // namespace ni

using namespace ni;

// ================================================================ C ABI

extern "C" int ni_inter_edges_workspace_size(int B, int H, int W, int connectivity, size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  const int64_t ne = int64_t(B) * H * W * (connectivity == 8 ? 4 : 2);
  Sizer z;
  z.take<int32_t>(ne);
  z.take<int32_t>(ne);
  z.take<char>(scan_ws_bytes(ne));
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_inter_edges(const int32_t* labels, const uint8_t* eflags, int B, int H, int W,
                              int connectivity, int32_t* keys_out, int32_t* n_out, void* workspace,
                              size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  const int kf = connectivity == 8 ? 4 : 2;
  const int64_t ne = npix * kf;
  NI_CHECK_ARG(ne < (int64_t(1) << 31), "too many edges for int32 keys");
  Carver c(workspace, workspace_bytes);
  int32_t* flag = c.take<int32_t>(ne);
  int32_t* pos = c.take<int32_t>(ne);
  void* sws = c.take<char>(scan_ws_bytes(ne));
  if (!c.ok() || !workspace) {
    set_error("ni_inter_edges: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), inter_flags_kernel<8><<<blocks_for(npix), 256, 0, s>>>(labels, eflags, W, npix, flag);
  else
    NI_COUNT_LAUNCH(), inter_flags_kernel<4><<<blocks_for(npix), 256, 0, s>>>(labels, eflags, W, npix, flag);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(flag, pos, ne, n_out, sws, s));
  NI_COUNT_LAUNCH(), compact_kernel<<<blocks_for(ne), 256, 0, s>>>(flag, pos, ne, keys_out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_quotient_workspace_size(int K, int count, size_t* bytes) {
  NI_CHECK_ARG(bytes && K >= 0 && count >= 0, "bad argument");
  Sizer z;
  Quot q;
  carve_quot(z, q, K, count);
  *bytes = z.used;
  return NI_OK;
}

// Static structure of the inter system for one partition (one map).
// SYNCHRONOUS (reads back the number of distinct component pairs).
extern "C" int ni_quotient_build(const int32_t* keys, int K, const int32_t* labels, int label_base,
                                 int count, int W, int connectivity, void* quot_ws,
                                 size_t quot_bytes, int32_t* n_pairs_host, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(K >= 0 && count >= 1, "bad sizes");
  NI_CHECK_ARG((int64_t)count * count < (int64_t(1) << 62), "too many components");
  cudaStream_t s = (cudaStream_t)stream;
  Carver c(quot_ws, quot_bytes);
  Quot q;
  carve_quot(c, q, K, count);
  if (!c.ok() || !quot_ws) {
    set_error("ni_quotient_build: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  const int C = count;
  if (K == 0) {
    NI_CUDA_TRY(cudaMemsetAsync(q.nU, 0, sizeof(int32_t), s));
    NI_CUDA_TRY(cudaMemsetAsync(q.cstart, 0, sizeof(int32_t) * (C + 1), s));
    NI_CUDA_TRY(cudaMemsetAsync(q.lstart, 0, sizeof(int32_t) * (C + 1), s));
    if (n_pairs_host) *n_pairs_host = 0;
    return NI_OK;
  }
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), quot_edges_kernel<8><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, label_base, W, C, q);
  else
    NI_COUNT_LAUNCH(), quot_edges_kernel<4><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, label_base, W, C, q);
  NI_LAUNCH_CHECK();
  const int pbits = end_bits_for((int64_t)C * C);
  size_t sb = q.sort_bytes;
  // (1) edges sorted by component pair (stable => edge order within a run)
  NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(q.sort_ws, sb, q.k64a, q.k64b, q.v32a, q.order, K, 0,
                                              pbits, s));
  NI_COUNT_LAUNCH(), run_flags_kernel<<<blocks_for(K), 256, 0, s>>>(q.k64b, K, q.flag);
  NI_LAUNCH_CHECK();
  // q.v32b holds incidence values; use q.lcol as scratch for run positions
  NI_TRY(exclusive_scan_i32(q.flag, q.lcol, K, q.nU, q.scan_ws, s));
  NI_COUNT_LAUNCH(), pair_runs_kernel<<<blocks_for(K), 256, 0, s>>>(q.k64b, K, C, q.lcol, q);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), set_tail_kernel<<<1, 1, 0, s>>>(q.pstart, q.nU, K);
  NI_LAUNCH_CHECK();
  // (2) incidence lists: (component, 2e+side) sorted by component, stable
  // keys are in q.flag? rebuild them (flag was overwritten by run flags)
  {
    if (connectivity == 8)
      NI_COUNT_LAUNCH(), quot_edges_kernel<8><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, label_base, W, C, q);
    else
      NI_COUNT_LAUNCH(), quot_edges_kernel<4><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, label_base, W, C, q);
    NI_LAUNCH_CHECK();
    const int cbits = end_bits_for(C);
    sb = q.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(q.sort_ws, sb, q.flag, q.v32a, q.v32b, q.cent,
                                                2 * K, 0, cbits, s));
    NI_CUDA_TRY(cudaMemsetAsync(q.hist, 0, sizeof(int32_t) * (C + 1), s));
    NI_COUNT_LAUNCH(), hist_kernel<<<blocks_for(2 * int64_t(K)), 256, 0, s>>>(q.flag, 2 * K, q.hist);
    NI_LAUNCH_CHECK();
    NI_TRY(exclusive_scan_i32(q.hist, q.cstart, C + 1, nullptr, q.scan_ws, s));
  }
  int32_t U = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&U, q.nU, sizeof(U), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  // (3) Laplacian sparsity: entries (row, col) for both directions of a pair
  NI_COUNT_LAUNCH(), lap_entries_kernel<<<blocks_for(U), 256, 0, s>>>(q, q.nU);
  NI_LAUNCH_CHECK();
  sb = q.sort_bytes;
  NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(q.sort_ws, sb, q.k64a, q.k64b, q.v32a, q.lpair, 2 * U,
                                              0, pbits, s));
  NI_COUNT_LAUNCH(), lap_cols_kernel<<<blocks_for(2 * int64_t(U)), 256, 0, s>>>(q, q.k64b, 2 * U);
  NI_LAUNCH_CHECK();
  NI_CUDA_TRY(cudaMemsetAsync(q.hist, 0, sizeof(int32_t) * (C + 1), s));
  NI_COUNT_LAUNCH(), hist_kernel<<<blocks_for(2 * int64_t(U)), 256, 0, s>>>(q.flag, 2 * U, q.hist);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(q.hist, q.lstart, C + 1, nullptr, q.scan_ws, s));
  if (n_pairs_host) *n_pairs_host = U;
  return NI_OK;
}

extern "C" int ni_scale_step_workspace_size(int K, int count, size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  Sizer z;
  StepWs w;
  carve_step(z, w, K, count);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_scale_step(const void* quot_ws, size_t quot_bytes, int K, int count,
                             const int32_t* labels, int label_base, const double* omega_a,
                             const double* omega_b, const double* gamma, const uint8_t* eflags,
                             int B, int H, int W, int connectivity, int model, int map_index, int t,
                             int alignment_iters, int mode, double k, double outlier_low,
                             double outlier_high, double cg_tol, int cg_max_iters, double* z,
                             double* scales, double* residual, double* weights, double* energy_out,
                             int32_t* cg_ok_out, void* workspace, size_t workspace_bytes,
                             ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(count >= 1 && K >= 0, "bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  Carver cq(const_cast<void*>(quot_ws), quot_bytes);
  Quot q;
  carve_quot(cq, q, K, count);
  Carver c(workspace, workspace_bytes);
  StepWs w;
  carve_step(c, w, K, count);
  if (!c.ok() || !workspace || !cq.ok()) {
    set_error("ni_scale_step: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  const int C = count;
  const int64_t npix = int64_t(B) * H * W;
  if (K == 0) {  // solver.py:293-295
    NI_COUNT_LAUNCH(), zero_kernel<<<blocks_for(C), 256, 0, s>>>(scales, C);
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemsetAsync(energy_out, 0, sizeof(double), s));
    NI_COUNT_LAUNCH(), set_int_kernel<<<1, 1, 0, s>>>(cg_ok_out, 1);
    NI_LAUNCH_CHECK();
    return NI_OK;
  }
  const int uniform = t < alignment_iters;
  const double lt = log10(outlier_low), ut = log10(outlier_high);
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), weights_kernel<8, 0><<<blocks_for(K), 256, 0, s>>>(q, z, omega_a, omega_b, gamma, eflags, H, W,
                                                       npix, uniform, mode, k, lt, ut, outlier_high, w);
  else if (model == 0)
    NI_COUNT_LAUNCH(), weights_kernel<4, 0><<<blocks_for(K), 256, 0, s>>>(q, z, omega_a, omega_b, gamma, eflags, H, W,
                                                       npix, uniform, mode, k, lt, ut, outlier_high, w);
  else
    NI_COUNT_LAUNCH(), weights_kernel<4, 1><<<blocks_for(K), 256, 0, s>>>(q, z, omega_a, omega_b, gamma, eflags, H, W,
                                                       npix, uniform, mode, k, lt, ut, outlier_high, w);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), pair_sum_kernel<<<blocks_for(32 * int64_t(K)), 256, 0, s>>>(q, w, q.nU);
  NI_CUDA_TRY(cudaMemsetAsync(w.anyflag, 0, sizeof(int32_t), s));
  NI_COUNT_LAUNCH(), comp_sum_kernel<<<blocks_for(32 * int64_t(C)), 256, 0, s>>>(q, w);
  NI_LAUNCH_CHECK();
  int32_t any = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&any, w.anyflag, sizeof(any), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  if (!any) {  // solver.py:112-113
    NI_COUNT_LAUNCH(), zero_kernel<<<blocks_for(C), 256, 0, s>>>(w.s, C);
    NI_LAUNCH_CHECK();
    NI_COUNT_LAUNCH(), set_int_kernel<<<1, 1, 0, s>>>(w.okflag, 1);
  } else {
    // remove the roundoff null-space component of A^T W b
    NI_COUNT_LAUNCH(), part_init_kernel<<<blocks_for(C), 256, 0, s>>>(w, C);
    NI_COUNT_LAUNCH(), part_union_kernel<<<blocks_for(K), 256, 0, s>>>(q, w, q.nU);
    NI_COUNT_LAUNCH(), part_flatten_kernel<<<blocks_for(C), 256, 0, s>>>(w, C);
    NI_LAUNCH_CHECK();
    size_t sb = w.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_ws, sb, w.pkey, w.pkey_s, w.pval, w.pval_s, C,
                                                0, end_bits_for(C), s));
    NI_COUNT_LAUNCH(), part_mean_kernel<<<blocks_for(32 * int64_t(C)), 256, 0, s>>>(w, C);
    NI_COUNT_LAUNCH(), part_sub_kernel<<<blocks_for(C), 256, 0, s>>>(w, C);
    NI_LAUNCH_CHECK();
    // K6
    int dev = 0;
    NI_CUDA_TRY(cudaGetDevice(&dev));
    int per_sm = 0;
    NI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scale_cg_kernel, kCgThreads, 0));
    int sms = 0;
    NI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int G = div_up(C, 4 * kCgThreads);
    const int gmax = per_sm * sms;
    if (G > gmax) G = gmax;
    if (G > kSMs) G = kSMs;
    if (G < 1) G = 1;
    const int maxiter = cg_max_iters > C ? cg_max_iters : C;
    double rtol = cg_tol;
    void* args[] = {&q, &w, &rtol, (void*)&maxiter};
    NI_COUNT_LAUNCH();
    NI_CUDA_TRY(cudaLaunchCooperativeKernel((void*)scale_cg_kernel, dim3(G), dim3(kCgThreads), args, 0,
                                            s));
  }
  NI_COUNT_LAUNCH(), residual_kernel<<<kResBlocks, 256, 0, s>>>(q, w, scales, residual, weights);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), energy_final_kernel<<<blocks_for(C), 256, 0, s>>>(w, kResBlocks, scales, C, energy_out, cg_ok_out);
  NI_LAUNCH_CHECK();
  const int64_t per_map = int64_t(H) * W;
  NI_COUNT_LAUNCH(), apply_kernel<<<blocks_for(per_map), 256, 0, s>>>(z, labels, w.s, label_base, map_index * per_map,
                                                   (map_index + 1) * per_map);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_merge_workspace_size(int K, int count, size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  Sizer z;
  MergeWs m;
  carve_merge(z, m, K, count);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_merge(const void* quot_ws, size_t quot_bytes, int K, int count, int32_t* labels,
                        int label_base, int H, int W, int map_index, const double* residual,
                        const double* weights, int32_t* new_count_out, double* energy_out,
                        void* workspace, size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(K >= 1 && count >= 1, "merge needs inter edges and components");
  cudaStream_t s = (cudaStream_t)stream;
  Carver cq(const_cast<void*>(quot_ws), quot_bytes);
  Quot q;
  carve_quot(cq, q, K, count);
  Carver c(workspace, workspace_bytes);
  MergeWs m;
  carve_merge(c, m, K, count);
  if (!c.ok() || !workspace || !cq.ok()) {
    set_error("ni_merge: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  const int C = count;
  NI_COUNT_LAUNCH(), merge_select_kernel<<<blocks_for(32 * int64_t(C)), 256, 0, s>>>(q, residual, m);
  NI_COUNT_LAUNCH(), merge_union_kernel<<<blocks_for(C), 256, 0, s>>>(q, m);
  NI_COUNT_LAUNCH(), merge_flatten_kernel<<<blocks_for(C), 256, 0, s>>>(m, C);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(m.flag, m.rank, C, m.total, m.scan_ws, s));
  NI_COUNT_LAUNCH(), merge_energy_kernel<<<kResBlocks, 256, 0, s>>>(q, m, residual, weights);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), merge_final_kernel<<<1, 1, 0, s>>>(m, kResBlocks, energy_out, new_count_out);
  NI_LAUNCH_CHECK();
  const int64_t per_map = int64_t(H) * W;
  NI_COUNT_LAUNCH(), merge_relabel_kernel<<<blocks_for(per_map), 256, 0, s>>>(labels, m, label_base,
                                                           map_index * per_map,
                                                           (map_index + 1) * per_map);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

// K4-K8: the relative-scale loop over the quotient graph, for a whole batch
// of maps at once.
//
//  * ni_inter_edges      graph.py:186-196   ordered compaction of inter edges
//  * ni_keys_filter      graph.py:186-196   the same, incrementally (after a
//                                           merge / when maps leave the loop)
//  * ni_quotient_build   solver.py:153-180  static structure of the pair system
//                                           (pair runs, component incidence,
//                                           Laplacian sparsity, per-map edge
//                                           ranges) of the batch's partition
//  * ni_scale_step       solver.py:253-303  weights (K4), segmented pair sums
//                                           (K5), one CG per map (K6),
//                                           residuals + per-map energy, z +=
//                                           s[label] (K7, pipeline.py:181-182)
//  * ni_merge            graph.py:207-250 + pipeline.py:187-203  (K8)
//
// Component ids are the batch's global labels: map m owns [first[m],
// first[m] + count[m]) (first[] fixed, count[] shrinking with merges); no
// edge, pair or part ever spans two maps, so the batch system is block
// diagonal and every per-map quantity (CG scalars, energy, merge ranks) is a
// segmented reduction.  Every floating-point sum runs in a fixed order (runs
// sorted by edge index, one block per map for per-map sums), so reruns are
// bit-identical and independent of which other maps share the batch.
#include <cooperative_groups.h>

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <vector>

#include "ni_common.cuh"
#include "ni_edges.cuh"

namespace cg = cooperative_groups;

namespace ni {

constexpr double kEnergyFloor = 1e-300;  // pipeline.py:55

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
  int K, C, B;
  int32_t* ea;        // [K] pixel a
  int32_t* eb;        // [K] pixel b
  int32_t* ek;        // [K] direction
  int32_t* pa;        // [K] component of a (global id, 0..C-1)
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
  int32_t* estart;    // [B+1] edges of map m: [estart[m], estart[m+1]) (keys are map-major)
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

static void carve_quot(Carver& c, Quot& q, int K, int C, int B) {
  const int64_t K2 = 2 * int64_t(K) + 1;
  q.K = K;
  q.C = C;
  q.B = B;
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
  q.estart = c.take<int32_t>(B + 1);
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
                                  const int32_t* __restrict__ labels, int W, int C, Quot q) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K; e += gridDim.x * blockDim.x) {
    const int32_t key = keys[e];
    const int32_t a = key / KF, k = key % KF;
    const int32_t b = a + fwd_dv(CONN, k) * W + fwd_du(CONN, k);
    const int32_t la = labels[a], lb = labels[b];
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

// Per-map edge ranges: keys are ascending pixel-edge ids, map-major.
__global__ void edge_ranges_kernel(const int32_t* __restrict__ keys, int K, int B,
                                   int64_t keys_per_map, int32_t* __restrict__ estart) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m > B) return;
  const int64_t target = int64_t(m) * keys_per_map;
  int lo = 0, hi = K;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (int64_t(keys[mid]) < target) lo = mid + 1;
    else hi = mid;
  }
  estart[m] = lo;
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

// Keep inter keys of kept maps whose endpoints carry different labels.
template <int CONN>
__global__ void keys_flag_kernel(const int32_t* __restrict__ keys, int K,
                                 const int32_t* __restrict__ labels,
                                 const uint8_t* __restrict__ map_keep, int64_t per_map, int W,
                                 int32_t* __restrict__ flag) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K; e += gridDim.x * blockDim.x) {
    const int32_t key = keys[e];
    const int32_t a = key / KF, k = key % KF;
    const int32_t b = a + fwd_dv(CONN, k) * W + fwd_du(CONN, k);
    flag[e] = map_keep[a / per_map] && labels[a] != labels[b];
  }
}

__global__ void keys_compact_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ flag,
                                    const int32_t* __restrict__ pos, int K,
                                    int32_t* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K; e += gridDim.x * blockDim.x)
    if (flag[e]) out[pos[e]] = keys[e];
}

// ------------------------------------------------------------ scale step

// Per-map tables, copied from the host into the workspace each call.
struct Maps {
  int B, nact;
  int32_t* first;   // [B+1]
  int32_t* count;   // [B]
  int32_t* active;  // [nact] maps taking part in this call
  const int32_t* live = nullptr;  // [B] device flags (nullable): a 0 makes the map sit the call out
};

__device__ __forceinline__ bool map_live(const Maps& mp, int m) { return !mp.live || mp.live[m]; }

// The three tables are one block of the workspace so that a call uploads
// them with ONE host->device copy (a pageable copy costs the stream ~10 us, and
// behind a bulk upload of the serving stream far more; the outer loop makes
// one call per iteration).
static void carve_maps(Carver& c, Maps& mp, int B) {
  mp.B = B;
  mp.first = c.take<int32_t>(3 * size_t(B + 1));
  mp.count = mp.first ? mp.first + (B + 1) : nullptr;
  mp.active = mp.first ? mp.first + 2 * (B + 1) : nullptr;
}

static int upload_maps(Maps& mp, const int32_t* first, const int32_t* count, const int32_t* active,
                       int nact, cudaStream_t s) {
  mp.nact = nact;
  const int B1 = mp.B + 1;
  static thread_local std::vector<int32_t> pack;
  pack.assign(3 * size_t(B1), 0);
  std::copy(first, first + B1, pack.begin());
  std::copy(count, count + mp.B, pack.begin() + B1);
  if (nact > 0) std::copy(active, active + nact, pack.begin() + 2 * B1);
  // pageable source: the driver stages it before the call returns
  NI_CUDA_TRY(cudaMemcpyAsync(mp.first, pack.data(), sizeof(int32_t) * (2 * B1 + nact),
                              cudaMemcpyHostToDevice, s));
  return NI_OK;
}

struct StepWs {
  double *wa, *wb, *ba, *bb, *S, *diag, *rhs, *r, *p0, *p1, *q, *part, *epart;
  int32_t *parent, *pkey, *pkey_s, *pval, *pval_s;
  int32_t* arrivals;  // [B] per-map block arrivals of residual_kernel
  Maps mp;
  void* sort_ws;
  size_t sort_bytes;
};

constexpr int kCgThreads = 512;
constexpr int kEChunks = 32;  // chunks of a map's edge range in per-map energies
constexpr int kBlockCgMax = 8192;  // maps up to this many components: one CTA each

static void carve_step(Carver& c, StepWs& w, int K, int C, int B) {
  w.wa = c.take<double>(K + 1);
  w.wb = c.take<double>(K + 1);
  w.ba = c.take<double>(K + 1);
  w.bb = c.take<double>(K + 1);
  w.S = c.take<double>(K + 1);
  w.diag = c.take<double>(C + 1);
  w.rhs = c.take<double>(C + 1);
  w.r = c.take<double>(C + 1);
  w.p0 = c.take<double>(C + 1);
  w.p1 = c.take<double>(C + 1);
  w.q = c.take<double>(C + 1);
  w.part = c.take<double>(4 * kSMs + 8);
  w.epart = c.take<double>(int64_t(B) * kEChunks);
  w.parent = c.take<int32_t>(C + 1);
  w.pkey = c.take<int32_t>(C + 1);
  w.pkey_s = c.take<int32_t>(C + 1);
  w.pval = c.take<int32_t>(C + 1);
  w.pval_s = c.take<int32_t>(C + 1);
  w.arrivals = c.take<int32_t>(B + 1);
  carve_maps(c, w.mp, B);
  w.sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, w.sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, C + 1);
  w.sort_ws = c.take<char>(w.sort_bytes);
}

// K4: weights and row right-hand sides (solver.py:253-278, 170-180)
template <int CONN, int MODEL>
__global__ void weights_kernel(Quot q, const double* __restrict__ z,
                               const double* __restrict__ zs, const int32_t* __restrict__ zlab,
                               const double* __restrict__ omega_a,
                               const double* __restrict__ omega_b,
                               const double* __restrict__ gamma,
                               const uint8_t* __restrict__ eflags, int H, int W, int64_t npix,
                               WeightArgs wp, StepWs w) {
  // grid.y = active map: only the edges of maps still in the loop
  const int m = w.mp.active[blockIdx.y];
  const int e1 = q.estart[m + 1];
  const bool live = map_live(w.mp, m);
  for (int e = q.estart[m] + blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += gridDim.x * blockDim.x) {
    if (!live) {  // a map that converged inside a chunk: its pair system stays zero
      w.wa[e] = w.wb[e] = w.ba[e] = w.bb[e] = 0.0;
      continue;
    }
    const int32_t a = q.ea[e], b = q.eb[e], k = q.ek[e];
    double wa, wb;
    edge_weights_at<CONN, MODEL>(z, zs, zlab, omega_a, omega_b, gamma, eflags, H, W, npix, a, k,
                                 wp, wa, wb);
    const double za = z_at(z, zs, zlab, a), zb = z_at(z, zs, zlab, b);
    const double oa = omega_a[k * npix + a];
    const double ob = MODEL == 0 ? -oa : omega_b[k * npix + a];
    w.wa[e] = wa;
    w.wb[e] = wb;
    w.ba[e] = oa - (za - zb);
    w.bb[e] = ob - (zb - za);
  }
}

// Strided segmented sums with the loads of kSumDepth consecutive steps in
// flight: a thread's gather chain (index -> operands) is two dependent L2
// round trips per step, so a serial loop is latency-bound (measured: a
// 1,500-edge pair cost one warp ~28 us).  The additions run in the same order
// as the plain loop, so the sums are bit-identical to it.  The operand arrays
// are not __restrict__: the fused kernel writes them earlier in the same
// launch, so they must not go through the non-coherent load path.
constexpr int kSumDepth = 8;

// sum of wa[e] + wb[e] over e = order[j], j = j0 + lane, + stride, ... < j1
__device__ __forceinline__ double run_pair_sum(const int32_t* __restrict__ order,
                                               const double* wa, const double* wb, int j,
                                               int j1, int stride) {
  double sum = 0.0;
  for (; j + (kSumDepth - 1) * stride < j1; j += kSumDepth * stride) {
    int e[kSumDepth];
    double a[kSumDepth], b[kSumDepth];
#pragma unroll
    for (int k = 0; k < kSumDepth; ++k) e[k] = order[j + k * stride];
#pragma unroll
    for (int k = 0; k < kSumDepth; ++k) {
      a[k] = wa[e[k]];
      b[k] = wb[e[k]];
    }
#pragma unroll
    for (int k = 0; k < kSumDepth; ++k) sum += a[k] + b[k];
  }
  for (; j < j1; j += stride) {
    const int e = order[j];
    sum += wa[e] + wb[e];
  }
  return sum;
}

// diagonal d and right-hand side r of a component over its incident entries
// cent[j], j = j0 + lane, + stride, ... < j1 (solver.py:108-111)
__device__ __forceinline__ void run_comp_sum(const int32_t* __restrict__ cent,
                                             const double* wa, const double* wb,
                                             const double* ba, const double* bb, int j, int j1,
                                             int stride, double& d, double& r) {
  constexpr int D = kSumDepth / 2;
  d = 0.0;
  r = 0.0;
  for (; j + (D - 1) * stride < j1; j += D * stride) {
    int ent[D];
    double va[D], vb[D], xa[D], xb[D];
#pragma unroll
    for (int k = 0; k < D; ++k) ent[k] = cent[j + k * stride];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int e = ent[k] >> 1;
      va[k] = wa[e];
      vb[k] = wb[e];
      xa[k] = ba[e];
      xb[k] = bb[e];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double t = va[k] * xa[k] - vb[k] * xb[k];
      d += va[k] + vb[k];
      r += (ent[k] & 1) ? -t : t;
    }
  }
  for (; j < j1; j += stride) {
    const int en = cent[j];
    const int e = en >> 1;
    const double a = wa[e], b = wb[e];
    const double t = a * ba[e] - b * bb[e];
    d += a + b;
    r += (en & 1) ? -t : t;
  }
}

// K5a + K5b in one launch (solver.py:108-111): blocks [0, pair_blocks) sum
// the conductance of each component pair over its run in edge order (a warp
// per pair, lane-strided + fixed xor tree), the others the diagonal and
// A^T W b of each component over its incident edges in edge order (a block
// per component); both reduction orders are independent of the grid.
__global__ void __launch_bounds__(256) sums_kernel(Quot q, StepWs w, const int32_t* __restrict__ nU_dev,
                                                   int pair_blocks) {
  __shared__ double red[32];
  if (int(blockIdx.x) < pair_blocks) {
    const int U = nU_dev[0];
    const int lane = threadIdx.x & 31;
    const int warps = (pair_blocks * blockDim.x) >> 5;
    for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += warps) {
      double sum = run_pair_sum(q.order, w.wa, w.wb, q.pstart[u] + lane, q.pstart[u + 1], 32);
      sum = warp_sum(sum);
      if (lane == 0) w.S[u] = sum;
    }
    return;
  }
  const int nb = gridDim.x - pair_blocks;
  for (int c = blockIdx.x - pair_blocks; c < q.C; c += nb) {
    double d, r;
    run_comp_sum(q.cent, w.wa, w.wb, w.ba, w.bb, q.cstart[c] + threadIdx.x, q.cstart[c + 1],
                 blockDim.x, d, r);
    d = block_sum(d, red);
    r = block_sum(r, red);
    if (threadIdx.x == 0) {
      w.diag[c] = d;
      w.rhs[c] = r;
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

// maps of <= kWarpMaxComps components project their right-hand side inside
// the CG kernel (one warp), so this pass leaves them alone: a map's arithmetic
// never depends on which other maps share the batch
constexpr int kWarpMaxComps = 32;

__device__ __forceinline__ int map_of_comp(const Maps& mp, int c) {
  int lo = 0, hi = mp.B - 1;  // last m with first[m] <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (mp.first[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void part_sub_kernel(StepWs w, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    if (w.mp.count[map_of_comp(w.mp, c)] > kWarpMaxComps) w.rhs[c] = w.rhs[c] - w.r[c];
}

// K6: scipy-equivalent CG on one map's component Laplacian (solver.py:97-122):
// x0 = 0, stop when ||r|| < rtol ||b|| at the top of an iteration, at most
// maxiter = max(cg_max_iters, C_m) iterations.  Rows [c0, c1) are the map's
// components; its Laplacian never references another map's columns.
struct CgArgs {
  int c0, c1, maxiter;
  double rtol;
  double* s;     // the map's scales (global id space)
  int32_t* ok;   // the map's "converged" flag
  int map;       // the map (cooperative launches: checked against the live flags)
};

// apply the Laplacian to p = r + beta pold for rows [c0, c1) with stride
template <class Sum>
__device__ __forceinline__ double cg_sweep(const Quot& q, const StepWs& w, const CgArgs& g,
                                           int tid, int stride, double beta, const double* pold,
                                           double* pnew) {
  double pq = 0.0;
  for (int c = g.c0 + tid; c < g.c1; c += stride) {
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
  return pq;
}

// scipy's CG from x0 = 0 (solver.py:97-122) for a map of n <= 32 components,
// one warp, a lane per component: the lane's Laplacian row (diagonal dg,
// off-diagonal conductances s_cnd[.][lane] at lanes s_col[.][lane], deg of
// them, jmax = the warp's largest deg) and right-hand side b; neighbours' p
// by shuffle, the iteration's three dots in one set of shuffle rounds
// (<r',r'> = <r,r> - 2 a <r,q> + a^2 <q,q>).  Returns the lane's x.
__device__ __forceinline__ double warp_cg(int lane, bool own, int deg, int jmax, double dg,
                                          double b, int n, double rtol, int cg_max_iters,
                                          const int8_t (*s_col)[32], const double (*s_cnd)[32],
                                          int& ok) {
  const int maxiter = cg_max_iters > n ? cg_max_iters : n;
  double x = 0.0, r = b, pv = 0.0;
  double rr = warp_sum(b * b);
  const double bnrm = sqrt(rr);
  ok = 1;
  if (bnrm == 0.0) return 0.0;
  const double atol = rtol * bnrm;
  double rho_prev = 0.0;
  ok = 0;
  // the first four row entries in registers: their shuffles of p are
  // independent, so they issue back to back instead of one shared-memory
  // round trip + shuffle per entry (the iteration is one long latency chain)
  int col4[4];
  double cnd4[4];
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    col4[jj] = jj < deg ? int(s_col[jj][lane]) : lane;
    cnd4[jj] = jj < deg ? s_cnd[jj][lane] : 0.0;
  }
  for (int it = 0; it < maxiter; ++it) {
    const double rho = rr;
    // (the division is issued beside the square root of the stop test)
    const double beta = it == 0 ? 0.0 : rho / rho_prev;
    if (sqrt(rr) < atol) {
      ok = 1;
      break;
    }
    pv = r + beta * pv;
    double aq = dg * pv;
    double pn4[4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
      if (jj < jmax) pn4[jj] = __shfl_sync(0xffffffffu, pv, col4[jj]);  // jmax is warp-uniform
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
      if (jj < deg) aq -= cnd4[jj] * pn4[jj];
    for (int jj = 4; jj < jmax; ++jj) {
      const bool has = jj < deg;
      const double pn = __shfl_sync(0xffffffffu, pv, has ? int(s_col[jj][lane]) : lane);
      if (has) aq -= s_cnd[jj][lane] * pn;
    }
    double d0 = pv * aq, d1 = r * aq, d2 = aq * aq;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d0 += __shfl_xor_sync(0xffffffffu, d0, o);
      d1 += __shfl_xor_sync(0xffffffffu, d1, o);
      d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    }
    const double alpha = rho / d0;
    x += alpha * pv;
    r -= alpha * aq;
    rr = fmax(rho - 2.0 * alpha * d1 + alpha * alpha * d2, 0.0);
    rho_prev = rho;
  }
  return own ? x : 0.0;
}

// the lane's Laplacian row of a small map into shared memory; returns its
// length, jmax = the warp's largest
__device__ __forceinline__ int warp_rows(const Quot& q, const StepWs& w, int c0, int lane,
                                         bool own, int8_t (*s_col)[32], double (*s_cnd)[32],
                                         int& jmax) {
  const int c = c0 + lane;
  const int j0 = own ? q.lstart[c] : 0, deg = own ? q.lstart[c + 1] - j0 : 0;
  for (int jj = 0; jj < deg; ++jj) {
    s_col[jj][lane] = int8_t(q.lcol[j0 + jj] - c0);
    s_cnd[jj][lane] = w.S[q.lpair[j0 + jj]];
  }
  __syncwarp();
  jmax = deg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
  return deg;
}

// the right-hand side minus its mean over the lane's part (the components
// joined by positive-conductance links: min-label propagation, < 32 rounds)
__device__ __forceinline__ double warp_project(int lane, bool own, int deg, int jmax, int n,
                                               double b0, const int8_t (*s_col)[32],
                                               const double (*s_cnd)[32]) {
  int part = own ? lane : 32 + lane;
  for (int round = 0; round < 32; ++round) {
    int nl = part;
    for (int jj = 0; jj < jmax; ++jj) {  // every lane takes part in every shuffle
      const bool link = jj < deg && s_cnd[jj][lane] > 0.0;
      const int other = __shfl_sync(0xffffffffu, part, link ? int(s_col[jj][lane]) : lane);
      if (link) nl = min(nl, other);
    }
    const bool changed = nl != part;
    part = nl;
    if (!__any_sync(0xffffffffu, changed)) break;
  }
  double psum = 0.0, pcnt = 0.0;
  for (int l = 0; l < n; ++l) {
    const int pl = __shfl_sync(0xffffffffu, part, l);
    const double bl = __shfl_sync(0xffffffffu, b0, l);
    if (pl == part) {
      psum += bl;
      pcnt += 1.0;
    }
  }
  return own ? b0 - psum / pcnt : 0.0;
}

// One CTA per map (maps with <= kBlockCgMax components): every reduction is
// a block reduction, so the whole solve runs without a grid barrier.
__global__ void __launch_bounds__(kCgThreads) scale_cg_block_kernel(Quot q, StepWs w, double rtol,
                                                                    int cg_max_iters, double* s,
                                                                    int32_t* ok_out) {
  __shared__ double red[32];
  const int m = w.mp.active[blockIdx.x];
  const int c0 = w.mp.first[m], n = w.mp.count[m], c1 = c0 + n;
  if (n > kBlockCgMax || !map_live(w.mp, m)) return;  // cooperative kernel / sitting out
  if (n <= kWarpMaxComps) {  // one warp, a lane per component: projection + CG
    __shared__ int8_t s_col[32][32];
    __shared__ double s_cnd[32][32];
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const bool own = lane < n;
    int jmax;
    const int deg = warp_rows(q, w, c0, lane, own, s_col, s_cnd, jmax);
    const double b = warp_project(lane, own, deg, jmax, n, own ? w.rhs[c0 + lane] : 0.0, s_col,
                                  s_cnd);
    if (own) w.rhs[c0 + lane] = b;
    int ok;
    const double x = warp_cg(lane, own, deg, jmax, own ? w.diag[c0 + lane] : 0.0, b, n, rtol,
                             cg_max_iters, s_col, s_cnd, ok);
    if (own) s[c0 + lane] = x;
    if (lane == 0) ok_out[m] = ok;
    return;
  }
  const int tid = threadIdx.x, stride = blockDim.x;
  const int maxiter = cg_max_iters > n ? cg_max_iters : n;
  double rr = 0.0;
  for (int c = c0 + tid; c < c1; c += stride) {
    const double b = w.rhs[c];
    s[c] = 0.0;
    w.r[c] = b;
    w.p0[c] = 0.0;
    rr += b * b;
  }
  rr = block_sum(rr, red);
  const double bnrm = sqrt(rr);
  if (bnrm == 0.0) {
    if (tid == 0) ok_out[m] = 1;
    return;
  }
  const double atol = rtol * bnrm;
  double rho_prev = 0.0;
  double* pold = w.p0;
  double* pnew = w.p1;
  int ok = 0;
  CgArgs g{c0, c1, maxiter, rtol, s, ok_out, m};
  for (int it = 0; it < maxiter; ++it) {
    if (sqrt(rr) < atol) {
      ok = 1;
      break;
    }
    const double rho = rr;
    const double beta = it == 0 ? 0.0 : rho / rho_prev;
    __syncthreads();  // every thread's reads of the previous r / pold are done
    double pq = cg_sweep<int>(q, w, g, tid, stride, beta, pold, pnew);
    pq = block_sum(pq, red);
    const double alpha = rho / pq;
    double rn = 0.0;
    for (int c = c0 + tid; c < c1; c += stride) {
      s[c] += alpha * pnew[c];
      const double r2 = w.r[c] - alpha * w.q[c];
      w.r[c] = r2;
      rn += r2 * r2;
    }
    rr = block_sum(rn, red);
    rho_prev = rho;
    double* t = pold;
    pold = pnew;
    pnew = t;
  }
  if (tid == 0) ok_out[m] = ok;
}

// Maps with more components: one cooperative launch per map; every block
// redundantly sums the per-block partials in block order, so all blocks
// agree bit for bit on every scalar.
__device__ __forceinline__ double grid_sum(cg::grid_group& grid, double v, double* part, int slot,
                                           double* red) {
  v = block_sum(v, red);
  if (threadIdx.x == 0) part[slot * gridDim.x + blockIdx.x] = v;
  grid.sync();
  double t = 0.0;
  for (int b = 0; b < int(gridDim.x); ++b) t += __ldcg(part + slot * gridDim.x + b);
  return t;
}

__global__ void __launch_bounds__(kCgThreads) scale_cg_kernel(Quot q, StepWs w, CgArgs g) {
  if (!map_live(w.mp, g.map)) return;  // uniform over the grid: before any grid sync
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  const int tid0 = g.c0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  double rr = 0.0;
  for (int c = tid0; c < g.c1; c += stride) {
    const double b = w.rhs[c];
    g.s[c] = 0.0;
    w.r[c] = b;
    w.p0[c] = 0.0;
    rr += b * b;
  }
  rr = grid_sum(grid, rr, w.part, 0, red);
  const double bnrm = sqrt(rr);
  if (bnrm == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) g.ok[0] = 1;
    return;
  }
  const double atol = g.rtol * bnrm;
  double rho_prev = 0.0;
  double* pold = w.p0;
  double* pnew = w.p1;
  int ok = 0;
  for (int it = 0; it < g.maxiter; ++it) {
    if (sqrt(rr) < atol) {
      ok = 1;
      break;
    }
    const double rho = rr;
    const double beta = it == 0 ? 0.0 : rho / rho_prev;
    double pq = cg_sweep<int>(q, w, g, tid0 - g.c0, stride, beta, pold, pnew);
    pq = grid_sum(grid, pq, w.part, 1, red);
    const double alpha = rho / pq;
    double rn = 0.0;
    for (int c = tid0; c < g.c1; c += stride) {
      g.s[c] += alpha * pnew[c];
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
  if (blockIdx.x == 0 && threadIdx.x == 0) g.ok[0] = ok;
}

// K7a: residual rows and the per-map energy (solver.py:301-302); one CTA
// per map over the map's edge range, in edge order.
// Per-map sums over edge ranges, split in kEChunks contiguous chunks (one
// block each, blockIdx.y = the map's slot in the active list) whose partials
// are added in chunk order: a fixed order independent of the batch.

__device__ __forceinline__ void chunk_range(int e0, int e1, int& c0, int& c1) {
  const int len = (e1 - e0 + kEChunks - 1) / kEChunks;
  c0 = min(e1, e0 + int(blockIdx.x) * len);
  c1 = min(e1, c0 + len);
}

__global__ void chunk_sum_kernel(const double* __restrict__ part, const int32_t* __restrict__ maps,
                                 int n, double* __restrict__ out,
                                 const int32_t* __restrict__ live) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || (live && !live[maps[j]])) return;
  double e = 0.0;
  for (int c = 0; c < kEChunks; ++c) e += part[j * kEChunks + c];
  out[maps[j]] = e;
}

// K7a + the per-map energy + the deferred shift in one launch: a map's
// kEChunks blocks write their partial energies; the last to finish (a
// per-map arrival counter) sums them in chunk order (as chunk_sum_kernel);
// each block also adds its share of the map's scales to zshift.
__global__ void __launch_bounds__(256) residual_kernel(Quot q, StepWs w, const double* __restrict__ s,
                                                       double* __restrict__ residual,
                                                       double* __restrict__ weights,
                                                       double* __restrict__ part,
                                                       double* __restrict__ energy_out,
                                                       int32_t* __restrict__ arrivals,
                                                       double* __restrict__ zshift) {
  __shared__ double red[32];
  __shared__ bool last;
  const int m = w.mp.active[blockIdx.y];
  if (!map_live(w.mp, m)) return;
  if (zshift) {  // zshift[c] += s[c] over this block's share of the map's components
    const int cf = w.mp.first[m], cn = w.mp.count[m];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cn; j += gridDim.x * blockDim.x)
      zshift[cf + j] += s[cf + j];
  }
  int c0, c1;
  chunk_range(q.estart[m], q.estart[m + 1], c0, c1);
  double en = 0.0;
  for (int e = c0 + threadIdx.x; e < c1; e += blockDim.x) {
    const double sa = s[q.pa[e]], sb = s[q.pb[e]];
    const double ra = sa - sb - w.ba[e];
    const double rb = sb - sa - w.bb[e];
    residual[2 * e] = ra;
    residual[2 * e + 1] = rb;
    weights[2 * e] = w.wa[e];
    weights[2 * e + 1] = w.wb[e];
    en += ra * (w.wa[e] * ra) + rb * (w.wb[e] * rb);
  }
  en = block_sum(en, red);
  if (threadIdx.x == 0) {
    part[blockIdx.y * kEChunks + blockIdx.x] = en;
    __threadfence();
    last = atomicAdd(arrivals + blockIdx.y, 1) == kEChunks - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double e = 0.0;
    for (int c = 0; c < kEChunks; ++c) e += __ldcg(part + blockIdx.y * kEChunks + c);
    energy_out[m] = e;
    arrivals[blockIdx.y] = 0;  // ready for the next call on this workspace
  }
}

// K7b: z[valid] += s[label] on the active maps' pixels (pipeline.py:181-182)
// grid.y = active map; U independent label/scale/z chains per thread.
__global__ void apply_kernel(double* __restrict__ z, const int32_t* __restrict__ labels,
                             const double* __restrict__ s, const int32_t* __restrict__ active,
                             int64_t per_map, const int32_t* __restrict__ live = nullptr) {
  constexpr int U = 4;
  if (live && !live[active[blockIdx.y]]) return;
  const int64_t base = int64_t(active[blockIdx.y]) * per_map;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j0 < per_map;
       j0 += U * stride) {
    int32_t l[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      l[u] = j < per_map ? labels[base + j] : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (l[u] >= 0) z[base + j0 + u * stride] += s[l[u]];
  }
}

// zshift[label] = 0 for every labelled pixel of the listed maps (after the
// shift was applied to z)
__global__ void shift_clear_kernel(double* __restrict__ zshift, const int32_t* __restrict__ labels,
                                   const int32_t* __restrict__ maps, int64_t per_map) {
  const int64_t base = int64_t(maps[blockIdx.y]) * per_map;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < per_map;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int32_t l = labels[base + j];
    if (l >= 0) zshift[l] = 0.0;
  }
}

__global__ void set_ok_kernel(int32_t* __restrict__ ok, const int32_t* __restrict__ active, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) ok[active[j]] = 1;
}

__global__ void zero_map_kernel(double* __restrict__ energy, const int32_t* __restrict__ active,
                                int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) energy[active[j]] = 0.0;
}

// ----------------------------------------------------------------- merge

struct MergeWs {
  double* epart;
  int32_t *sel, *parent, *flag, *rank, *cmap;
  uint8_t* merging;  // [B]
  Maps mp;
  void* scan_ws;
};

static void carve_merge(Carver& c, MergeWs& m, int K, int C, int B) {
  m.epart = c.take<double>(int64_t(B) * kEChunks);
  m.sel = c.take<int32_t>(C + 1);
  m.parent = c.take<int32_t>(C + 1);
  m.flag = c.take<int32_t>(C + 2);
  m.rank = c.take<int32_t>(C + 2);
  m.cmap = c.take<int32_t>(C + 1);
  m.merging = c.take<uint8_t>(B + 1);
  carve_maps(c, m.mp, B);
  m.scan_ws = c.take<char>(scan_ws_bytes(C + 2));
}

// map of every live component id (-1: id above its map's current count)
__global__ void comp_map_kernel(MergeWs m, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    int lo = 0, hi = m.mp.B;  // last map with first <= c
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (m.mp.first[mid] <= c) lo = mid;
      else hi = mid;
    }
    m.cmap[c] = c < m.mp.first[lo] + m.mp.count[lo] ? lo : -1;
  }
}

__global__ void merging_flags_kernel(MergeWs m) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= m.mp.B; j += gridDim.x * blockDim.x)
    m.merging[j] = 0;
}

__global__ void merging_set_kernel(MergeWs m) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m.mp.nact) m.merging[m.mp.active[j]] = 1;
}

// argmin over incident inter edges of (|residual_a|, edge index)
// (graph.py:230-239); one warp per component of a merging map,
// lexicographic warp argmin.
__global__ void merge_select_kernel(Quot q, const double* __restrict__ residual, MergeWs m) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < q.C; c += warps) {
    const int mc = m.cmap[c];
    int best_e = -1;
    double best = 0.0;
    if (mc >= 0 && m.merging[mc]) {
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
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= C; c += gridDim.x * blockDim.x) {
    if (c == C) {
      m.flag[C] = 0;
      continue;
    }
    const int r = uf_find(m.parent, c);
    m.parent[c] = r;
    m.flag[c] = r == c && m.cmap[c] >= 0;
  }
}

// new count of every map (unchanged for maps that do not merge)
__global__ void merge_counts_kernel(MergeWs m, int32_t* __restrict__ new_count) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m.mp.B; j += gridDim.x * blockDim.x) {
    const int f = m.mp.first[j];
    new_count[j] = m.rank[f + m.mp.count[j]] - m.rank[f];
  }
}

__global__ void merge_relabel_kernel(int32_t* __restrict__ labels, const MergeWs m, int64_t per_map,
                                     int64_t n) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int mm = m.mp.active[j / per_map];
    const int64_t i = int64_t(mm) * per_map + j % per_map;
    const int32_t l = labels[i];
    if (l >= 0) {
      const int f = m.mp.first[mm];
      labels[i] = f + m.rank[m.parent[l]] - m.rank[f];
    }
  }
}

// energy restricted to edges that stay inter-component (pipeline.py:196-203);
// one CTA per merging map, in edge order
__global__ void __launch_bounds__(256) merge_energy_kernel(Quot q, const MergeWs m,
                                                           const double* __restrict__ residual,
                                                           const double* __restrict__ weights,
                                                           double* __restrict__ part) {
  __shared__ double red[32];
  const int mm = m.mp.active[blockIdx.y];
  int c0, c1;
  chunk_range(q.estart[mm], q.estart[mm + 1], c0, c1);
  double en = 0.0;
  for (int e = c0 + threadIdx.x; e < c1; e += blockDim.x) {
    if (m.parent[q.pa[e]] != m.parent[q.pb[e]]) {
      const double ra = residual[2 * e], rb = residual[2 * e + 1];
      en += ra * (weights[2 * e] * ra) + rb * (weights[2 * e + 1] * rb);
    }
  }
  en = block_sum(en, red);
  if (threadIdx.x == 0) part[blockIdx.y * kEChunks + blockIdx.x] = en;
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

extern "C" int ni_keys_filter_workspace_size(int K, size_t* bytes) {
  NI_CHECK_ARG(bytes && K >= 0, "bad argument");
  Sizer z;
  z.take<int32_t>(K + 1);
  z.take<int32_t>(K + 1);
  z.take<char>(scan_ws_bytes(K + 1));
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_keys_filter(const int32_t* keys, int K, const int32_t* labels,
                              const uint8_t* map_keep, int H, int W, int connectivity,
                              int32_t* keys_out, int32_t* n_out, void* workspace,
                              size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(K >= 0 && keys_out != keys, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  Carver c(workspace, workspace_bytes);
  int32_t* flag = c.take<int32_t>(K + 1);
  int32_t* pos = c.take<int32_t>(K + 1);
  void* sws = c.take<char>(scan_ws_bytes(K + 1));
  if (!c.ok() || !workspace) {
    set_error("ni_keys_filter: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  if (K == 0) {
    NI_CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(int32_t), s));
    return NI_OK;
  }
  const int64_t per_map = int64_t(H) * W;
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), keys_flag_kernel<8><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, map_keep,
                                                                       per_map, W, flag);
  else
    NI_COUNT_LAUNCH(), keys_flag_kernel<4><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, map_keep,
                                                                       per_map, W, flag);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(flag, pos, K, n_out, sws, s));
  NI_COUNT_LAUNCH(), keys_compact_kernel<<<blocks_for(K), 256, 0, s>>>(keys, flag, pos, K, keys_out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_quotient_workspace_size(int K, int count, int B, size_t* bytes) {
  NI_CHECK_ARG(bytes && K >= 0 && count >= 0 && B >= 1, "bad argument");
  Sizer z;
  Quot q;
  carve_quot(z, q, K, count, B);
  *bytes = z.used;
  return NI_OK;
}

// Static structure of the inter system of the batch's partition.
// SYNCHRONOUS (reads back the number of distinct component pairs and, if
// map_edges_host is given, the B per-map edge counts).
extern "C" int ni_quotient_build(const int32_t* keys, int K, const int32_t* labels, int count,
                                 int B, int H, int W, int connectivity, void* quot_ws,
                                 size_t quot_bytes, int32_t* n_pairs_host, int32_t* map_edges_host,
                                 ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(K >= 0 && count >= 1 && B >= 1, "bad sizes");
  NI_CHECK_ARG((int64_t)count * count < (int64_t(1) << 62), "too many components");
  cudaStream_t s = (cudaStream_t)stream;
  Carver c(quot_ws, quot_bytes);
  Quot q;
  carve_quot(c, q, K, count, B);
  if (!c.ok() || !quot_ws) {
    set_error("ni_quotient_build: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  const int C = count;
  const int kf = connectivity == 8 ? 4 : 2;
  NI_COUNT_LAUNCH(), edge_ranges_kernel<<<div_up(B + 1, 128), 128, 0, s>>>(
                         keys, K, B, int64_t(H) * W * kf, q.estart);
  NI_LAUNCH_CHECK();
  int32_t U = 0;
  if (K == 0) {
    NI_CUDA_TRY(cudaMemsetAsync(q.nU, 0, sizeof(int32_t), s));
    NI_CUDA_TRY(cudaMemsetAsync(q.cstart, 0, sizeof(int32_t) * (C + 1), s));
    NI_CUDA_TRY(cudaMemsetAsync(q.lstart, 0, sizeof(int32_t) * (C + 1), s));
  } else {
    if (connectivity == 8)
      NI_COUNT_LAUNCH(), quot_edges_kernel<8><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, W, C, q);
    else
      NI_COUNT_LAUNCH(), quot_edges_kernel<4><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, W, C, q);
    NI_LAUNCH_CHECK();
    const int pbits = end_bits_for((int64_t)C * C);
    size_t sb = q.sort_bytes;
    // (1) edges sorted by component pair (stable => edge order within a run)
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(q.sort_ws, sb, q.k64a, q.k64b, q.v32a, q.order, K,
                                                0, pbits, s));
    NI_COUNT_LAUNCH(), run_flags_kernel<<<blocks_for(K), 256, 0, s>>>(q.k64b, K, q.flag);
    NI_LAUNCH_CHECK();
    // q.lcol as scratch for run positions
    NI_TRY(exclusive_scan_i32(q.flag, q.lcol, K, q.nU, q.scan_ws, s));
    NI_COUNT_LAUNCH(), pair_runs_kernel<<<blocks_for(K), 256, 0, s>>>(q.k64b, K, C, q.lcol, q);
    NI_LAUNCH_CHECK();
    NI_COUNT_LAUNCH(), set_tail_kernel<<<1, 1, 0, s>>>(q.pstart, q.nU, K);
    NI_LAUNCH_CHECK();
    // (2) incidence lists: (component, 2e+side) sorted by component, stable
    // (the incidence keys in q.flag were overwritten by the run flags)
    if (connectivity == 8)
      NI_COUNT_LAUNCH(), quot_edges_kernel<8><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, W, C, q);
    else
      NI_COUNT_LAUNCH(), quot_edges_kernel<4><<<blocks_for(K), 256, 0, s>>>(keys, K, labels, W, C, q);
    NI_LAUNCH_CHECK();
    const int cbits = end_bits_for(C);
    sb = q.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(q.sort_ws, sb, q.flag, q.v32a, q.v32b, q.cent,
                                                2 * K, 0, cbits, s));
    NI_CUDA_TRY(cudaMemsetAsync(q.hist, 0, sizeof(int32_t) * (C + 1), s));
    NI_COUNT_LAUNCH(), hist_kernel<<<blocks_for(2 * int64_t(K)), 256, 0, s>>>(q.flag, 2 * K, q.hist);
    NI_LAUNCH_CHECK();
    NI_TRY(exclusive_scan_i32(q.hist, q.cstart, C + 1, nullptr, q.scan_ws, s));
    NI_CUDA_TRY(cudaMemcpyAsync(&U, q.nU, sizeof(U), cudaMemcpyDeviceToHost, s));
    NI_CUDA_TRY(cudaStreamSynchronize(s));
    // (3) Laplacian sparsity: entries (row, col) for both directions of a pair
    NI_COUNT_LAUNCH(), lap_entries_kernel<<<blocks_for(U), 256, 0, s>>>(q, q.nU);
    NI_LAUNCH_CHECK();
    sb = q.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(q.sort_ws, sb, q.k64a, q.k64b, q.v32a, q.lpair,
                                                2 * U, 0, pbits, s));
    NI_COUNT_LAUNCH(), lap_cols_kernel<<<blocks_for(2 * int64_t(U)), 256, 0, s>>>(q, q.k64b, 2 * U);
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemsetAsync(q.hist, 0, sizeof(int32_t) * (C + 1), s));
    NI_COUNT_LAUNCH(), hist_kernel<<<blocks_for(2 * int64_t(U)), 256, 0, s>>>(q.flag, 2 * U, q.hist);
    NI_LAUNCH_CHECK();
    NI_TRY(exclusive_scan_i32(q.hist, q.lstart, C + 1, nullptr, q.scan_ws, s));
  }
  if (map_edges_host) {
    std::vector<int32_t> es(B + 1);
    NI_CUDA_TRY(cudaMemcpyAsync(es.data(), q.estart, sizeof(int32_t) * (B + 1),
                                cudaMemcpyDeviceToHost, s));
    NI_CUDA_TRY(cudaStreamSynchronize(s));
    for (int m = 0; m < B; ++m) map_edges_host[m] = es[m + 1] - es[m];
  }
  if (n_pairs_host) *n_pairs_host = U;
  return NI_OK;
}

extern "C" int ni_scale_step_workspace_size(int K, int count, int B, size_t* bytes) {
  NI_CHECK_ARG(bytes && K >= 0 && count >= 0 && B >= 1, "bad argument");
  Sizer z;
  StepWs w;
  carve_step(z, w, K, count, B);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_scale_step(const void* quot_ws, size_t quot_bytes, int K, int count, int B,
                             const int32_t* map_first, const int32_t* map_count,
                             const int32_t* active, int nact, const int32_t* labels,
                             const double* omega_a, const double* omega_b, const double* gamma,
                             const uint8_t* eflags, int H, int W, int connectivity, int model, int t,
                             int alignment_iters, int mode, double k, double outlier_low,
                             double outlier_high, double cg_tol, int cg_max_iters, double* z,
                             double* zshift, const int32_t* live, double* scales,
                             double* residual, double* weights, double* energy_out,
                             int32_t* cg_ok_out, void* workspace, size_t workspace_bytes,
                             ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(count >= 1 && K >= 0 && B >= 1 && nact >= 0 && nact <= B, "bad sizes");
  NI_CHECK_ARG(map_first && map_count && (active || nact == 0), "null map table");
  cudaStream_t s = (cudaStream_t)stream;
  Carver cq(const_cast<void*>(quot_ws), quot_bytes);
  Quot q;
  carve_quot(cq, q, K, count, B);
  Carver c(workspace, workspace_bytes);
  StepWs w;
  carve_step(c, w, K, count, B);
  if (!c.ok() || !workspace || !cq.ok()) {
    set_error("ni_scale_step: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  if (nact == 0) return NI_OK;
  NI_TRY(upload_maps(w.mp, map_first, map_count, active, nact, s));
  w.mp.live = live;
  const int C = count;
  const int64_t npix = int64_t(B) * H * W;
  if (K == 0) {  // solver.py:293-295: no inter edge anywhere in the batch
    NI_COUNT_LAUNCH(), zero_map_kernel<<<div_up(nact, 128), 128, 0, s>>>(energy_out, w.mp.active, nact);
    NI_COUNT_LAUNCH(), set_ok_kernel<<<div_up(nact, 128), 128, 0, s>>>(cg_ok_out, w.mp.active, nact);
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemsetAsync(scales, 0, sizeof(double) * C, s));
    return NI_OK;
  }
  if (nact < B) {
    // maps that left the loop keep their edges in the quotient; the pair and
    // component sums read every edge, so theirs must hold zeros, not stale
    // workspace (the active maps' systems are block-diagonal from them)
    NI_CUDA_TRY(cudaMemsetAsync(w.wa, 0, sizeof(double) * K, s));
    NI_CUDA_TRY(cudaMemsetAsync(w.wb, 0, sizeof(double) * K, s));
    NI_CUDA_TRY(cudaMemsetAsync(w.ba, 0, sizeof(double) * K, s));
    NI_CUDA_TRY(cudaMemsetAsync(w.bb, 0, sizeof(double) * K, s));
  }
  WeightArgs wp;
  wp.wmode = t < alignment_iters ? EW_UNIFORM : EW_FULL;
  wp.mode = mode;
  wp.k = k;
  wp.lt = log10(outlier_low);
  wp.ut = log10(outlier_high);
  wp.hi = outlier_high;
  // one thread per inter edge, all in flight: each edge's weight gathers a
  // few scattered pixels (latency-bound with fewer threads)
  const dim3 wblocks(unsigned(std::max<int64_t>(
                         1, std::min<int64_t>((int64_t(K) / std::max(B, 1) + 255) / 256 + 1,
                                              int64_t(kSMs) * 64 / nact + 1))),
                     unsigned(nact));
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), weights_kernel<8, 0><<<wblocks, 256, 0, s>>>(
                           q, z, zshift, labels, omega_a, omega_b, gamma, eflags, H, W, npix, wp, w);
  else if (model == 0)
    NI_COUNT_LAUNCH(), weights_kernel<4, 0><<<wblocks, 256, 0, s>>>(
                           q, z, zshift, labels, omega_a, omega_b, gamma, eflags, H, W, npix, wp, w);
  else
    NI_COUNT_LAUNCH(), weights_kernel<4, 1><<<wblocks, 256, 0, s>>>(
                           q, z, zshift, labels, omega_a, omega_b, gamma, eflags, H, W, npix, wp, w);
  NI_LAUNCH_CHECK();
  {
    const int pb = blocks_for(32 * int64_t(K));
    const int cb = int(std::min<int64_t>(C, int64_t(kSMs) * 8));
    NI_COUNT_LAUNCH(), sums_kernel<<<pb + cb, 256, 0, s>>>(q, w, q.nU, pb);
  }
  NI_LAUNCH_CHECK();
  // remove the roundoff null-space component of A^T W b; maps
  // of <= kWarpMaxComps components do it in their CG warp
  bool any_big = false;
  for (int j = 0; j < nact; ++j) any_big |= map_count[active[j]] > kWarpMaxComps;
  if (any_big) {
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
  }
  // K6: one CTA per map, and one cooperative launch per large map
  NI_COUNT_LAUNCH(), scale_cg_block_kernel<<<nact, kCgThreads, 0, s>>>(q, w, cg_tol, cg_max_iters,
                                                                      scales, cg_ok_out);
  NI_LAUNCH_CHECK();
  int G = 0;
  for (int j = 0; j < nact; ++j) {
    const int m = active[j];
    const int n = map_count[m];
    if (n <= kBlockCgMax) continue;
    if (G == 0) {
      int dev = 0, per_sm = 0, sms = 0;
      NI_CUDA_TRY(cudaGetDevice(&dev));
      NI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scale_cg_kernel, kCgThreads, 0));
      NI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      G = per_sm * sms < kSMs ? per_sm * sms : kSMs;
    }
    int g = div_up(n, 4 * kCgThreads);
    if (g > G) g = G;
    if (g < 1) g = 1;
    CgArgs ca{map_first[m], map_first[m] + n, cg_max_iters > n ? cg_max_iters : n, cg_tol, scales,
              cg_ok_out + m, m};
    void* args[] = {&q, &w, &ca};
    NI_COUNT_LAUNCH();
    NI_CUDA_TRY(cudaLaunchCooperativeKernel((void*)scale_cg_kernel, dim3(g), dim3(kCgThreads), args,
                                            0, s));
  }
  NI_CUDA_TRY(cudaMemsetAsync(w.arrivals, 0, sizeof(int32_t) * nact, s));
  NI_COUNT_LAUNCH(), residual_kernel<<<dim3(kEChunks, nact), 256, 0, s>>>(
                         q, w, scales, residual, weights, w.epart, energy_out, w.arrivals, zshift);
  NI_LAUNCH_CHECK();
  const int64_t per_map = int64_t(H) * W;
  if (!zshift) {
    const int bx = int(std::max<int64_t>(
        1, std::min<int64_t>((per_map + 1023) / 1024, int64_t(kSMs) * 16 / nact + 1)));
    NI_COUNT_LAUNCH(), apply_kernel<<<dim3(bx, nact), 256, 0, s>>>(z, labels, scales,
                                                                  w.mp.active, per_map, live);
  }
  NI_LAUNCH_CHECK();
  return NI_OK;
}

// ---------------------------------------------------- fused per-map step
//
// Maps whose quotient is small (<= kFusedMaxEdges inter edges, <=
// kFusedMaxComps components) take the whole iteration -- weights, pair and
// component sums, the null-space projection, the CG, residual rows, energy,
// the deferred shift and the convergence test -- in ONE CTA: one launch per
// iteration for every such map of the batch instead of ~15 small launches.
// Same arithmetic as the multi-kernel step; the pair sums, component sums
// and CG reduce in the same orders, the part means and the energy in other
// fixed orders (a map's path depends only on its own sizes, so batched and
// single-map runs stay bit-identical).
constexpr int kFusedThreads = 512;
#ifndef NI_FUSED_MAX_EDGES
#define NI_FUSED_MAX_EDGES (1 << 14)  // measured: 64 C5 maps (~50 k edges each) run faster as
#endif                                // the multi-kernel step spread over every SM (51.9 ms per
                                      // step against 53.5 ms with a cluster per map)
constexpr int kFusedMaxEdges = NI_FUSED_MAX_EDGES;
constexpr int kFusedMaxComps = 1024;
#ifndef NI_FUSED_CLUSTER
#define NI_FUSED_CLUSTER 8  // CTAs per map (a thread-block cluster; 8 is the portable maximum)
#endif
constexpr int kFusedCluster = NI_FUSED_CLUSTER;
static_assert(kFusedCluster >= 1 && kFusedCluster <= 8, "portable cluster sizes only");

struct DecideArgs {
  int t;  // 1-based iteration after this step
  int max_iters, alignment_iters;
  double delta_e_max;
  double* e_prev;
  int32_t* live;
  int32_t* iters;
  double* e_hist;
  int32_t* ok_hist;
  int hist_stride;
  int32_t* nlive;
};

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One outer iteration of map m by the whole CTA (the body of the chunk loop).
template <int CONN, int MODEL>
__device__ void fused_iteration(
    int m, const Quot& q, const StepWs& w, const double* __restrict__ z,
    const double* zs, const int32_t* __restrict__ zlab,
    const double* __restrict__ omega_a, const double* __restrict__ omega_b,
    const double* __restrict__ gamma, const uint8_t* __restrict__ eflags, int H, int W,
    int64_t npix, const WeightArgs& wp, double rtol, int cg_max_iters, double* __restrict__ s,
    double* __restrict__ residual, double* __restrict__ weights, double* __restrict__ energy_out,
    int32_t* __restrict__ ok_out, double* zshift, const DecideArgs& da, double* red) {
  __shared__ double s_cnd[32][32];  // small maps: entry j of lane's Laplacian row (<= 31)
  __shared__ int8_t s_col[32][32];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank()), CL = int(cl.num_blocks());
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int gtid = rank * nt + tid, gnt = CL * nt;  // thread / warp of the map's cluster
  const int gwid = rank * nw + wid, gnw = CL * nw;
  const int e0 = q.estart[m], e1 = q.estart[m + 1];
  const int c0 = w.mp.first[m], n = w.mp.count[m], c1 = c0 + n;
  // K4: weights and row right-hand sides (solver.py:253-278, 170-180); two
  // edges per step so their gather chains overlap (restrict copies let the
  // compiler hoist the second edge's loads over the first edge's stores)
  const int32_t* __restrict__ qea = q.ea;
  const int32_t* __restrict__ qeb = q.eb;
  const int32_t* __restrict__ qek = q.ek;
  double* __restrict__ wwa = w.wa;
  double* __restrict__ wwb = w.wb;
  double* __restrict__ wba = w.ba;
  double* __restrict__ wbb = w.bb;
#pragma unroll 2
  for (int e = e0 + gtid; e < e1; e += gnt) {
    const int32_t a = qea[e], b = qeb[e], k = qek[e];
    double wa, wb;
    edge_weights_at<CONN, MODEL>(z, zs, zlab, omega_a, omega_b, gamma, eflags, H, W, npix, a, k,
                                 wp, wa, wb);
    const double za = z_at(z, zs, zlab, a), zb = z_at(z, zs, zlab, b);
    const double oa = omega_a[k * npix + a];
    const double ob = MODEL == 0 ? -oa : omega_b[k * npix + a];
    wwa[e] = wa;
    wwb[e] = wb;
    wba[e] = oa - (za - zb);
    wbb[e] = ob - (zb - za);
  }
  cl.sync();
  // K5a: pair conductances (the map's pairs are a contiguous run of the
  // (min, max)-sorted pair list); a warp per pair, as sums_kernel
  const int U = q.nU[0];
  const int u0 = lower_bound_i32(q.pp, U, c0), u1 = lower_bound_i32(q.pp, U, c1);
  for (int u = u0 + gwid; u < u1; u += gnw) {
    double sum = run_pair_sum(q.order, w.wa, w.wb, q.pstart[u] + lane, q.pstart[u + 1], 32);
    sum = warp_sum(sum);
    if (lane == 0) w.S[u] = sum;
  }
  // K5b: diagonal and A^T W b per component: a warp per component (the
  // cluster's warps in reverse, so pairs and components start on different
  // ends), lane-strided over its incident entries in edge order
  for (int c = c0 + (gnw - 1 - gwid); c < c1; c += gnw) {
    double d, r;
    run_comp_sum(q.cent, w.wa, w.wb, w.ba, w.bb, q.cstart[c] + lane, q.cstart[c + 1], 32, d, r);
    d = warp_sum(d);
    r = warp_sum(r);
    if (lane == 0) {
      w.diag[c] = d;
      w.rhs[c] = r;
    }
  }
  cl.sync();  // every warp's pair sum, diagonal and right-hand side is written
  if (rank != 0) {
    // the solve is the first CTA's
  } else if (n <= 32) {
    // One warp, a lane per component: the parts (components joined by
    // S > 0) by label propagation, the roundoff null-space projection of the
    // right-hand side, and the CG.
    if (wid == 0) {
      const int c = c0 + lane;
      const bool own = lane < n;
      int jmax;
      const int deg = warp_rows(q, w, c0, lane, own, s_col, s_cnd, jmax);
      const double b = warp_project(lane, own, deg, jmax, n, own ? w.rhs[c] : 0.0, s_col, s_cnd);
      if (own) w.rhs[c] = b;
      int ok = 1;
      const double x = warp_cg(lane, own, deg, jmax, own ? w.diag[c] : 0.0, b, n, rtol,
                               cg_max_iters, s_col, s_cnd, ok);
      if (own) s[c] = x;
      if (lane == 0) ok_out[m] = ok;
    }
    __syncthreads();
  } else {
  // roundoff null-space removal per part (components joined by S > 0)
    for (int c = c0 + tid; c < c1; c += nt) w.parent[c] = c;
    __syncthreads();
    for (int u = u0 + tid; u < u1; u += nt)
      if (w.S[u] > 0.0) uf_union(w.parent, q.pp[u], q.pq[u]);
    __syncthreads();
    for (int c = c0 + tid; c < c1; c += nt) w.pkey[c] = uf_find(w.parent, c);
    __syncthreads();
    // a warp per part root: its components in ascending id, lane-strided
    for (int r0 = c0 + wid; r0 < c1; r0 += nw) {
      if (w.pkey[r0] != r0) continue;  // warp-uniform
      double sum = 0.0, cnt = 0.0;
      for (int c = c0 + lane; c < c1; c += 32)
        if (w.pkey[c] == r0) {
          sum += w.rhs[c];
          cnt += 1.0;
        }
      sum = warp_sum(sum);
      cnt = warp_sum(cnt);
      if (lane == 0) w.r[r0] = sum / cnt;  // the part's mean, stashed at its root
    }
    __syncthreads();
    for (int c = c0 + tid; c < c1; c += nt) w.q[c] = w.rhs[c] - w.r[w.pkey[c]];
    __syncthreads();
    for (int c = c0 + tid; c < c1; c += nt) w.rhs[c] = w.q[c];
    __syncthreads();
    const int maxiter = cg_max_iters > n ? cg_max_iters : n;
    double rr = 0.0;
    for (int c = c0 + tid; c < c1; c += nt) {
      const double b = w.rhs[c];
      s[c] = 0.0;
      w.r[c] = b;
      w.p0[c] = 0.0;
      rr += b * b;
    }
    rr = block_sum(rr, red);
    const double bnrm = sqrt(rr);
    int ok = 1;
    if (bnrm != 0.0) {
      const double atol = rtol * bnrm;
      double rho_prev = 0.0;
      double* pold = w.p0;
      double* pnew = w.p1;
      ok = 0;
      CgArgs g{c0, c1, maxiter, rtol, s, ok_out, m};
      for (int it = 0; it < maxiter; ++it) {
        if (sqrt(rr) < atol) {
          ok = 1;
          break;
        }
        const double rho = rr;
        const double beta = it == 0 ? 0.0 : rho / rho_prev;
        __syncthreads();
        double pq = cg_sweep<int>(q, w, g, tid, nt, beta, pold, pnew);
        pq = block_sum(pq, red);
        const double alpha = rho / pq;
        double rn = 0.0;
        for (int c = c0 + tid; c < c1; c += nt) {
          s[c] += alpha * pnew[c];
          const double r2 = w.r[c] - alpha * w.q[c];
          w.r[c] = r2;
          rn += r2 * r2;
        }
        rr = block_sum(rn, red);
        rho_prev = rho;
        double* tp = pold;
        pold = pnew;
        pnew = tp;
      }
    }
    if (tid == 0) ok_out[m] = ok;
  }
  cl.sync();
  // K7a: residual rows and the map's energy (solver.py:301-302): a partial
  // per CTA, summed in rank order by the first
  double en = 0.0;
  for (int e = e0 + gtid; e < e1; e += gnt) {
    const double sa = s[q.pa[e]], sb = s[q.pb[e]];
    const double ra = sa - sb - w.ba[e];
    const double rb = sb - sa - w.bb[e];
    residual[2 * e] = ra;
    residual[2 * e + 1] = rb;
    weights[2 * e] = w.wa[e];
    weights[2 * e + 1] = w.wb[e];
    en += ra * (w.wa[e] * ra) + rb * (w.wb[e] * rb);
  }
  en = block_sum(en, red);
  if (CL > 1) {
    if (tid == 0) w.epart[int64_t(m) * kEChunks + rank] = en;
    // K7b: deferred z += s[label]
    for (int c = c0 + gtid; c < c1; c += gnt) zshift[c] += s[c];
    cl.sync();
    if (rank == 0 && tid == 0) {
      en = 0.0;
      for (int r = 0; r < CL; ++r) en += w.epart[int64_t(m) * kEChunks + r];
    }
  } else {
    for (int c = c0 + tid; c < c1; c += nt) zshift[c] += s[c];
  }
  // the convergence test of pipeline.py:66-83
  if (rank == 0 && tid == 0) {
    energy_out[m] = en;
    const double ep = da.e_prev[m];
    const int t = da.t;
    da.e_hist[int64_t(m) * da.hist_stride + t - 1] = en;
    da.ok_hist[int64_t(m) * da.hist_stride + t - 1] = ok_out[m];
    bool conv;
    if (t >= da.max_iters || en <= kEnergyFloor) conv = true;
    else if (t <= da.alignment_iters + 1 || ep <= kEnergyFloor) conv = false;
    else conv = fabs(en - ep) / ep < da.delta_e_max;
    da.e_prev[m] = en;
    if (conv) {
      da.live[m] = 0;
      da.iters[m] = t;
      atomicSub(da.nlive, 1);
    }
  }
  cl.sync();  // the live flag, the shifts and the scales before the next iteration
}

// k outer iterations of each map (a CTA per map, its loop entirely inside the
// CTA: maps never interact), stopping at the map's convergence.
template <int CONN, int MODEL>
__global__ void __launch_bounds__(kFusedThreads) scale_fused_kernel(
    Quot q, StepWs w, const double* __restrict__ z, const double* zs,
    const int32_t* __restrict__ zlab, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int64_t npix, WeightArgs wp, int t0,
    int k, int alignment_iters, double rtol, int cg_max_iters, double* __restrict__ s,
    double* __restrict__ residual, double* __restrict__ weights,
    double* __restrict__ energy_out, int32_t* __restrict__ ok_out,
    double* zshift, DecideArgs da) {
  // zs and zshift are the same array (the shifts are read by the weights and
  // advanced at the end of every iteration): neither is __restrict__, so the
  // reads stay on the coherent path
  __shared__ double red[32];
  const int m = w.mp.active[blockIdx.x / cg::this_cluster().num_blocks()];
  for (int i = 0; i < k; ++i) {
    if (!da.live[m]) return;  // uniform: written by thread 0 before the previous barrier
    WeightArgs wi = wp;
    wi.wmode = t0 + i < alignment_iters ? EW_UNIFORM : EW_FULL;
    DecideArgs di = da;
    di.t = t0 + i + 1;
    fused_iteration<CONN, MODEL>(m, q, w, z, zs, zlab, omega_a, omega_b, gamma, eflags, H, W,
                                 npix, wi, rtol, cg_max_iters, s, residual, weights, energy_out,
                                 ok_out, zshift, di, red);
  }
}

extern "C" int ni_scale_step_fused(const void* quot_ws, size_t quot_bytes, int K, int count, int B,
                                   const int32_t* map_first, const int32_t* map_count,
                                   const int32_t* active, int nact, const int32_t* labels,
                                   const double* omega_a, const double* omega_b,
                                   const double* gamma, const uint8_t* eflags, int H, int W,
                                   int connectivity, int model, int t, int k_iters,
                                   int alignment_iters,
                                   int mode, double k, double outlier_low, double outlier_high,
                                   double cg_tol, int cg_max_iters, const double* z,
                                   double* zshift, double* scales, double* residual,
                                   double* weights, double* energy_out, int32_t* cg_ok_out,
                                   int max_iters, double delta_e_max, double* e_prev,
                                   int32_t* live, int32_t* iters, double* e_hist, int32_t* ok_hist,
                                   int hist_stride, int32_t* nlive, void* workspace,
                                   size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(count >= 1 && K >= 1 && B >= 1 && nact >= 0 && nact <= B, "bad sizes");
  NI_CHECK_ARG(map_first && map_count && (active || nact == 0), "null map table");
  NI_CHECK_ARG(z && zshift && live && e_prev && iters && e_hist && ok_hist && nlive, "null pointer");
  NI_CHECK_ARG(t >= 0 && k_iters >= 1 && t + k_iters <= hist_stride, "bad iteration range");
  cudaStream_t s = (cudaStream_t)stream;
  Carver cq(const_cast<void*>(quot_ws), quot_bytes);
  Quot q;
  carve_quot(cq, q, K, count, B);
  Carver c(workspace, workspace_bytes);
  StepWs w;
  carve_step(c, w, K, count, B);
  if (!c.ok() || !workspace || !cq.ok()) {
    set_error("ni_scale_step_fused: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  if (nact == 0) return NI_OK;
  for (int j = 0; j < nact; ++j) {
    const int mm = active[j];
    NI_CHECK_ARG(mm >= 0 && mm < B && map_count[mm] <= kFusedMaxComps, "map too large to fuse");
  }
  NI_TRY(upload_maps(w.mp, map_first, map_count, active, nact, s));
  w.mp.live = live;
  WeightArgs wp;
  wp.wmode = EW_FULL;  // per iteration in the kernel
  wp.mode = mode;
  wp.k = k;
  wp.lt = log10(outlier_low);
  wp.ut = log10(outlier_high);
  wp.hi = outlier_high;
  DecideArgs da{t + 1, max_iters, alignment_iters, delta_e_max, e_prev, live, iters,
                e_hist, ok_hist, hist_stride, nlive};
  const int64_t npix = int64_t(B) * H * W;
  // a thread-block cluster per map: kFusedCluster CTAs on as many SMs share the
  // map's edge loops and segmented sums, with cluster barriers between the
  // stages (no grid barrier: maps never interact)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(nact) * kFusedCluster);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kFusedCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const double* zs_arg = zshift;
#define NI_FUSED(CN, MD)                                                                       \
  launched = cudaLaunchKernelEx(&cfg, scale_fused_kernel<CN, MD>, q, w, z, zs_arg, labels,     \
                                omega_a, omega_b, gamma, eflags, H, W, npix, wp, t, k_iters,   \
                                alignment_iters, cg_tol, cg_max_iters, scales, residual,       \
                                weights, energy_out, cg_ok_out, zshift, da)
  cudaError_t launched;
  NI_COUNT_LAUNCH();
  if (connectivity == 8) NI_FUSED(8, 0);
  else if (model == 0) NI_FUSED(4, 0);
  else NI_FUSED(4, 1);
#undef NI_FUSED
  NI_CUDA_TRY(launched);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_scale_fused_limits(int* max_edges, int* max_comps) {
  const char* ov = NI_ENV_ONCE("NI_FUSED_MAX_EDGES");  // measurement knob
  if (max_edges) *max_edges = ov ? atoi(ov) : kFusedMaxEdges;
  if (max_comps) *max_comps = kFusedMaxComps;
  return NI_OK;
}

// pipeline.py:66-83 for every live map of the active list after the step at
// 1-based iteration t: record E_t and the CG flag, then the convergence test
// against the previous energy; a converged map drops its live flag.
__global__ void loop_decide_kernel(const double* __restrict__ energy,
                                   const int32_t* __restrict__ ok, const int32_t* __restrict__ active,
                                   int nact, int t, int max_iters, int alignment_iters,
                                   double delta_e_max, double* __restrict__ e_prev,
                                   int32_t* __restrict__ live, int32_t* __restrict__ iters,
                                   double* __restrict__ e_hist, int32_t* __restrict__ ok_hist,
                                   int hist_stride, int32_t* __restrict__ nlive) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nact) return;
  const int m = active[j];
  if (!live[m]) return;
  const double e = energy[m], ep = e_prev[m];
  e_hist[int64_t(m) * hist_stride + t - 1] = e;
  ok_hist[int64_t(m) * hist_stride + t - 1] = ok[m];
  bool conv;
  if (t >= max_iters || e <= kEnergyFloor) conv = true;
  else if (t <= alignment_iters + 1 || ep <= kEnergyFloor) conv = false;
  else conv = fabs(e - ep) / ep < delta_e_max;
  e_prev[m] = e;
  if (conv) {
    live[m] = 0;
    iters[m] = t;
    if (nlive) atomicSub(nlive, 1);
  }
}

extern "C" int ni_loop_decide(const double* energy, const int32_t* cg_ok, const int32_t* active,
                              int nact, int t, int max_iters, int alignment_iters,
                              double delta_e_max, double* e_prev, int32_t* live, int32_t* iters,
                              double* e_hist, int32_t* ok_hist, int hist_stride,
                              int32_t* nlive, ni_stream_t stream) {
  NI_CHECK_ARG(energy && cg_ok && e_prev && live && iters && e_hist && ok_hist, "null pointer");
  NI_CHECK_ARG(nact >= 0 && t >= 1 && t <= hist_stride, "bad iteration / sizes");
  NI_CHECK_ARG(active || nact == 0, "null active list");
  if (nact == 0) return NI_OK;
  NI_COUNT_LAUNCH(), loop_decide_kernel<<<div_up(nact, 128), 128, 0, (cudaStream_t)stream>>>(
                         energy, cg_ok, active, nact, t, max_iters, alignment_iters, delta_e_max,
                         e_prev, live, iters, e_hist, ok_hist, hist_stride, nlive);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_apply_shift(double* z, double* zshift, const int32_t* labels, int B, int H, int W,
                              const int32_t* maps, int nmaps, void* workspace,
                              size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(z && zshift && labels && B >= 1 && nmaps >= 0 && nmaps <= B, "bad argument");
  NI_CHECK_ARG(maps || nmaps == 0, "null map list");
  NI_CHECK_ARG(workspace && workspace_bytes >= sizeof(int32_t) * size_t(std::max(nmaps, 1)),
               "workspace too small");
  if (nmaps == 0) return NI_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* dmaps = static_cast<int32_t*>(workspace);
  NI_CUDA_TRY(cudaMemcpyAsync(dmaps, maps, sizeof(int32_t) * nmaps, cudaMemcpyHostToDevice, s));
  const int64_t per_map = int64_t(H) * W;
  const int bx = int(std::max<int64_t>(
      1, std::min<int64_t>((per_map + 1023) / 1024, int64_t(kSMs) * 16 / nmaps + 1)));
  NI_COUNT_LAUNCH(), apply_kernel<<<dim3(bx, nmaps), 256, 0, s>>>(z, labels, zshift, dmaps, per_map);
  NI_LAUNCH_CHECK();
  // the shift is now in z: clear it for every component (labels of these maps
  // are the only ones that index their entries)
  NI_COUNT_LAUNCH(), shift_clear_kernel<<<dim3(bx, nmaps), 256, 0, s>>>(zshift, labels, dmaps,
                                                                       per_map);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_merge_workspace_size(int K, int count, int B, size_t* bytes) {
  NI_CHECK_ARG(bytes && K >= 0 && count >= 0 && B >= 1, "bad argument");
  Sizer z;
  MergeWs m;
  carve_merge(z, m, K, count, B);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_merge(const void* quot_ws, size_t quot_bytes, int K, int count, int B,
                        const int32_t* map_first, const int32_t* map_count, const int32_t* merging,
                        int nmerge, int32_t* labels, int H, int W, const double* residual,
                        const double* weights, int32_t* new_count_out, double* energy_out,
                        void* workspace, size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(K >= 1 && count >= 1 && B >= 1 && nmerge >= 1 && nmerge <= B,
               "merge needs inter edges, components and merging maps");
  NI_CHECK_ARG(map_first && map_count && merging, "null map table");
  cudaStream_t s = (cudaStream_t)stream;
  Carver cq(const_cast<void*>(quot_ws), quot_bytes);
  Quot q;
  carve_quot(cq, q, K, count, B);
  Carver c(workspace, workspace_bytes);
  MergeWs m;
  carve_merge(c, m, K, count, B);
  if (!c.ok() || !workspace || !cq.ok()) {
    set_error("ni_merge: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  NI_TRY(upload_maps(m.mp, map_first, map_count, merging, nmerge, s));
  const int C = count;
  NI_COUNT_LAUNCH(), comp_map_kernel<<<blocks_for(C), 256, 0, s>>>(m, C);
  NI_COUNT_LAUNCH(), merging_flags_kernel<<<div_up(B + 1, 256), 256, 0, s>>>(m);
  NI_COUNT_LAUNCH(), merging_set_kernel<<<div_up(nmerge, 256), 256, 0, s>>>(m);
  NI_COUNT_LAUNCH(), merge_select_kernel<<<blocks_for(32 * int64_t(C)), 256, 0, s>>>(q, residual, m);
  NI_COUNT_LAUNCH(), merge_union_kernel<<<blocks_for(C), 256, 0, s>>>(q, m);
  NI_COUNT_LAUNCH(), merge_flatten_kernel<<<blocks_for(C + 1), 256, 0, s>>>(m, C);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(m.flag, m.rank, C + 1, nullptr, m.scan_ws, s));
  NI_COUNT_LAUNCH(), merge_counts_kernel<<<div_up(B, 256), 256, 0, s>>>(m, new_count_out);
  NI_COUNT_LAUNCH(), merge_energy_kernel<<<dim3(kEChunks, nmerge), 256, 0, s>>>(q, m, residual,
                                                                                 weights, m.epart);
  NI_COUNT_LAUNCH(), chunk_sum_kernel<<<div_up(nmerge, 64), 64, 0, s>>>(m.epart, m.mp.active,
                                                                       nmerge, energy_out, nullptr);
  NI_LAUNCH_CHECK();
  const int64_t per_map = int64_t(H) * W;
  NI_COUNT_LAUNCH(), merge_relabel_kernel<<<blocks_for(nmerge * per_map), 256, 0, s>>>(
                         labels, m, per_map, nmerge * per_map);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

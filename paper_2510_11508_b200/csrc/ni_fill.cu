// K3 -- fill_components (solver.py:195-239) as ONE batched CG over every
// component of the partition, matrix-free on the pixel grid, run by ONE
// persistent cooperative kernel whose workers are independent warps.
//
// Per component c the reference solves (A^T W A) x = A^T W b with scipy's
// unpreconditioned CG (x0 = 0, stop when ||r|| < rtol ||b|| at the top of an
// iteration, cap max(cg_max_iters, n_c); solver.py:97-122).  At the fill
// state z = 0 every bilateral factor is 1/2 (continuity.py:302-308), so
// W_a = gamma_a^2 / 2 and A^T W A is the graph Laplacian of the intra-
// component valid edges with conductance c_ab = W_a + W_b (SURVEY.md
// Appendix A).  All components iterate together; each keeps its own
// alpha/beta/rho, stop test and cap, exactly like separate scipy solves.
// The stencil is applied in difference form q_a = sum c_ab (p_a - p_b), so
// constants stay an exact null vector in float32 (a rounded CSR Laplacian
// loses that and doubles the iteration count).
//
// Data layout in HBM (per pixel, npix = B*H*W, row-major):
//   x             : float32 solution
//   r[2], q[2], p[2] : float32 CG vectors, double-buffered by iteration parity
//                   (a sweep reads its neighbours' previous values while
//                   other warps write the new ones)
//   hw            : float32 W_a = gamma_a^2 / 2  (c_ab = hw_a + hw_b)
//   imask         : uint8, bit k = forward edge k intra-component and valid,
//                   bit 4+k = backward edge k (pixel - offset_k)
//
// ONE sweep and ONE grid sync per CG iteration.  scipy's iteration k
//   p_k = r_k + beta p_{k-1};  q_k = A p_k;  alpha = rho_k / <p_k, q_k>;
//   x_{k+1} = x_k + alpha p_k;  r_{k+1} = r_k - alpha q_k;  rho_{k+1} = <r_{k+1}, r_{k+1}>
// is regrouped so that sweep k forms r_k = r_{k-1} - alpha_{k-1} q_{k-1} and
// x_k = x_{k-1} + alpha_{k-1} p_{k-1} on the fly (also for the stencil halo),
// then p_k and q_k, and reduces <p,q>, <r,q>, <q,q>, <r,r> in the same pass.
// rho_k = <r_k, r_k> is exact; rho_{k+1}, needed for beta and for scipy's
// stop test before r_{k+1} exists, is rho_k - 2 alpha <r,q> + alpha^2 <q,q>
// (float64, no cancellation at CG's per-step contraction).  A component that
// stops gets one last "flush" sweep that applies its pending x update.
//
// Work decomposition: the grid is cut into strips of 30 columns x 32 rows.
// A warp processes a strip by marching down its rows with a register ring
// of rows y-1, y, y+1 (+ prefetched rows); lanes 0 and 31 carry the left /
// right halo columns, so horizontal neighbours are warp shuffles and there
// is no block barrier anywhere in a sweep.  A strip touching several
// multi-pixel components becomes ceil(n/2) "items" of <= 2 components that
// read the int32 labels; a strip with one component (the common case) is a
// "pure" item that needs no label at all (singletons / invalid pixels carry
// r = q = p = 0 and stay 0 under any update).
//
// Reductions are deterministic: each item writes float64 partials per
// component (lane-local sums over rows, fixed xor tree over lanes); the last
// warp to arrive for a component (integer counter) sums the component's
// partials in plan order and updates its scalars.
// Algorithmic bytes per active pixel and iteration (pure items):
//   read r, q, p, x, hw (20 B) + imask (1 B); write r, q, p, x (16 B) => 37 B/px
// (halo rows/columns are re-read from L2 and not counted).
#include <cooperative_groups.h>
#include <stdlib.h>

#include <cub/device/device_radix_sort.cuh>

#include "ni_common.cuh"

namespace cg = cooperative_groups;

namespace ni {

constexpr int SW = 30;     // strip width (lanes 1..30)
constexpr int SH = 32;     // strip height (rows per item)
constexpr int SPX = 1024;  // padded pixels per strip (sort buffer)
constexpr int NT = 256;    // threads per CTA (8 warps)
constexpr int WPB = NT / 32;
constexpr int SLOTS = 2;  // components per item
constexpr int PF = 3;     // rows prefetched ahead
constexpr int NDOT = 4;   // <p,q>, <r,q>, <q,q>, <r,r>

enum : uint8_t { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_CAPPED = 2, ST_IDLE = 3, ST_FLUSH = 4 };

// One work item: a strip and up to 2 of its components.
struct __align__(16) Item {
  int32_t x0, y0;  // top-left pixel of the strip (column of lane 1)
  int32_t pbase;   // first partial slot of this item
  int32_t flags;   // bits 0-7: components in the item (1..2); bit 8: pure strip
  int32_t comp[SLOTS];
};

__device__ __forceinline__ int item_n(const Item& it) { return it.flags & 0xFF; }
__device__ __forceinline__ bool item_pure(const Item& it) { return (it.flags >> 8) & 1; }

struct FillArgs {
  int rows, W;
  float* x;
  float* r[2];
  float* q[2];
  float* p[2];
  const float* hw;
  const uint8_t* imask;
  const int32_t* labels;
  // plan
  const Item* items;
  int nitems;
  const int32_t* comp_pstart;  // [C+1] partial range per component
  const int32_t* comp_plist;   // [P] partial indices grouped by component
  int32_t* comp_cnt;           // [C] arrival counters (zero between sweeps)
  double* partial;             // [P][NDOT]
  int32_t* active_items;       // [2][nitems]
  int32_t* nactive_items;      // [2]
  // component state
  double* rho;     // exact <r_k, r_k> / then the rho_{k+1} estimate
  double* alpha;   // alpha of the last completed sweep
  double* beta;
  double* tol;
  int32_t* iters;
  int32_t* cap;
  uint8_t* status;
  uint8_t* final_status;  // status after the flush sweep
  int32_t* active;   // components still ACTIVE or FLUSH
  int32_t* changed;  // a component changed state during the last sweep
};

// ----------------------------------------------------------------- setup

template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) prep_kernel(
    const int32_t* __restrict__ labels, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int64_t npix, float* __restrict__ hw,
    uint8_t* __restrict__ imask, float* __restrict__ x, float* __restrict__ r,
    float* __restrict__ r1, float* __restrict__ q0, float* __restrict__ q1, float* __restrict__ p0,
    float* __restrict__ p1, int32_t* __restrict__ comp_size) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t lab = labels[i];
    x[i] = 0.f;
    r1[i] = 0.f;
    q0[i] = 0.f;
    q1[i] = 0.f;
    p0[i] = 0.f;
    p1[i] = 0.f;
    if (lab < 0) {
      hw[i] = 0.f;
      imask[i] = 0;
      r[i] = 0.f;
      continue;
    }
    atomicAdd(comp_size + lab, 1);
    const double wa = 0.5 * (gamma[i] * gamma[i]);
    hw[i] = float(wa);
    const int u = int(i % W);
    const int vloc = int((i / W) % H);
    const uint8_t ef = eflags[i];
    uint8_t m = 0;
    double b = 0.0;
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
      // forward edge (i -> j): the row centred at i is the "a" row
      if ((ef >> k) & (ef >> (4 + k)) & 1) {
        const int64_t j = i + int64_t(dv) * W + du;
        if (labels[j] == lab) {
          m |= uint8_t(1u << k);
          const double wb = 0.5 * (gamma[j] * gamma[j]);
          const double oa = omega_a[k * npix + i];
          const double ob = MODEL == 0 ? -oa : omega_b[k * npix + i];
          b += wa * oa - wb * ob;  // A^T W b of rows 2e, 2e+1 (solver.py:83-93)
        }
      }
      // backward edge (j -> i), j = i - offset_k: i is the "b" endpoint
      const int uj = u - du, vj = vloc - dv;
      if (uj >= 0 && uj < W && vj >= 0) {
        const int64_t j = i - int64_t(dv) * W - du;
        const uint8_t efj = eflags[j];
        if (((efj >> k) & (efj >> (4 + k)) & 1) && labels[j] == lab) {
          m |= uint8_t(1u << (4 + k));
          const double wj = 0.5 * (gamma[j] * gamma[j]);
          const double oa = omega_a[k * npix + j];
          const double ob = MODEL == 0 ? -oa : omega_b[k * npix + j];
          b += wa * ob - wj * oa;
        }
      }
    }
    imask[i] = m;
    r[i] = float(b);
  }
}

// One CTA per strip: its distinct multi-pixel components, ascending.
__global__ void __launch_bounds__(NT) strip_comps_kernel(const int32_t* __restrict__ labels,
                                                         const int32_t* __restrict__ comp_size,
                                                         int rows, int W, int nsx,
                                                         int32_t* __restrict__ nslots,
                                                         int32_t* __restrict__ strip_comps) {
  __shared__ int32_t key[SPX];
  __shared__ int32_t wcount[WPB];
  const int strip = blockIdx.x, tid = threadIdx.x;
  const int x0 = (strip % nsx) * SW, y0 = (strip / nsx) * SH;
  for (int e = tid; e < SPX; e += NT) {
    int32_t lab = -1;
    if (e < SW * SH) {
      const int gx = x0 + (e % SW), gy = y0 + (e / SW);
      if (gx < W && gy < rows) {
        lab = labels[int64_t(gy) * W + gx];
        if (lab >= 0 && comp_size[lab] < 2) lab = -1;  // singletons never iterate (solver.py:220)
      }
    }
    key[e] = lab < 0 ? INT32_MAX : lab;
  }
  __syncthreads();
  for (int k = 2; k <= SPX; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int e = tid; e < SPX; e += NT) {
        const int ixj = e ^ j;
        if (ixj > e) {
          const int32_t a = key[e], b = key[ixj];
          const bool up = (e & k) == 0;
          if ((a > b) == up) {
            key[e] = b;
            key[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  constexpr int PER = SPX / NT;
  int cnt = 0;
  bool first[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = tid * PER + j;
    first[j] = key[e] != INT32_MAX && (e == 0 || key[e - 1] != key[e]);
    cnt += first[j];
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if ((tid & 31) >= o) incl += t;
  }
  if ((tid & 31) == 31) wcount[tid >> 5] = incl;
  __syncthreads();
  int before = incl - cnt;
  for (int w = 0; w < (tid >> 5); ++w) before += wcount[w];
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (first[j]) strip_comps[int64_t(strip) * SPX + before++] = key[tid * PER + j];
  if (tid == NT - 1) nslots[strip] = before;
}

__global__ void strip_items_kernel(const int32_t* __restrict__ nslots,
                                   const int32_t* __restrict__ slot_base,
                                   const int32_t* __restrict__ item_base,
                                   const int32_t* __restrict__ strip_comps, int nstrips, int nsx,
                                   Item* __restrict__ items, int32_t* __restrict__ partial_comp,
                                   int32_t* __restrict__ partial_idx,
                                   int32_t* __restrict__ comp_nparts) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nstrips; s += gridDim.x * blockDim.x) {
    const int ns = nslots[s];
    if (ns == 0) continue;
    const int pb = slot_base[s], ib = item_base[s];
    for (int k = 0; k * SLOTS < ns; ++k) {
      Item it;
      it.x0 = (s % nsx) * SW;
      it.y0 = (s / nsx) * SH;
      it.pbase = pb + k * SLOTS;
      const int n = min(SLOTS, ns - k * SLOTS);
      it.flags = n | ((ns == 1 ? 1 : 0) << 8);
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        it.comp[j] = j < n ? strip_comps[int64_t(s) * SPX + k * SLOTS + j] : -1;
      items[ib + k] = it;
    }
    for (int j = 0; j < ns; ++j) {
      const int32_t c = strip_comps[int64_t(s) * SPX + j];
      partial_comp[pb + j] = c;
      partial_idx[pb + j] = pb + j;
      atomicAdd(comp_nparts + c, 1);
    }
  }
}

__global__ void item_counts_kernel(const int32_t* __restrict__ nslots, int nstrips,
                                   int32_t* __restrict__ nitems) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nstrips; s += gridDim.x * blockDim.x)
    nitems[s] = (nslots[s] + SLOTS - 1) / SLOTS;
}

// ------------------------------------------------------- warp machinery

__device__ __forceinline__ int slot_of(const Item& it, int32_t lab) {
  int s = -1;
  const int n = item_n(it);
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
    if (j < n && it.comp[j] == lab) s = j;
  return s;
}

// Write the item's per-component partials (NDOT each), count arrivals, and
// let the last arriving warp of a component reduce its partials in plan
// order and call fin(c, dots).
template <class Fin>
__device__ __forceinline__ void item_finish(const FillArgs& a, const Item& it,
                                            double (&acc)[SLOTS][NDOT], const bool* live, Fin fin) {
  const int lane = threadIdx.x & 31;
  const int n = item_n(it);
  double tot[SLOTS][NDOT];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int d = 0; d < NDOT; ++d) tot[s][d] = warp_sum(acc[s][d]);
  unsigned last = 0;
  if (lane < n) {
    int32_t c = it.comp[0];
    bool lv = live[0];
    double v[NDOT];
#pragma unroll
    for (int d = 0; d < NDOT; ++d) v[d] = tot[0][d];
#pragma unroll
    for (int s = 1; s < SLOTS; ++s)
      if (lane == s) {
        c = it.comp[s];
        lv = live[s];
#pragma unroll
        for (int d = 0; d < NDOT; ++d) v[d] = tot[s][d];
      }
    if (lv) {
      double* dst = a.partial + size_t(it.pbase + lane) * NDOT;
#pragma unroll
      for (int d = 0; d < NDOT; ++d) dst[d] = v[d];
      __threadfence();
      const int32_t np = a.comp_pstart[c + 1] - a.comp_pstart[c];
      if (atomicAdd(a.comp_cnt + c, 1) == np - 1) last = 1;
    }
  }
  unsigned lastmask = __ballot_sync(0xffffffffu, last);
  while (lastmask) {
    const int s = __ffs(lastmask) - 1;
    lastmask &= lastmask - 1;
    int32_t c = it.comp[0];
#pragma unroll
    for (int j = 1; j < SLOTS; ++j)
      if (s == j) c = it.comp[j];
    __threadfence();
    const int32_t q0 = a.comp_pstart[c], q1 = a.comp_pstart[c + 1];
    double sum[NDOT] = {0.0, 0.0, 0.0, 0.0};
    for (int j = q0 + lane; j < q1; j += 32) {
      const double* src = a.partial + size_t(a.comp_plist[j]) * NDOT;
#pragma unroll
      for (int d = 0; d < NDOT; ++d) sum[d] += __ldcg(src + d);
    }
#pragma unroll
    for (int d = 0; d < NDOT; ++d) sum[d] = warp_sum(sum[d]);
    if (lane == 0) {
      fin(c, sum);
      a.comp_cnt[c] = 0;
    }
    __syncwarp();
  }
}

// Per-slot coefficients of the item for this sweep.
struct Coefs {
  float al[SLOTS], be[SLOTS];
  uint8_t st[SLOTS];
};

__device__ __forceinline__ bool item_coefs(const FillArgs& a, const Item& it, Coefs& k) {
  bool any = false;
  const int n = item_n(it);
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) {
    k.al[j] = 0.f;
    k.be[j] = 0.f;
    k.st[j] = ST_IDLE;
    if (j < n) {
      const int32_t c = it.comp[j];
      k.st[j] = __ldcg(a.status + c);
      k.al[j] = float(__ldcg(a.alpha + c));
      k.be[j] = float(__ldcg(a.beta + c));
      any |= k.st[j] == ST_ACTIVE || k.st[j] == ST_FLUSH;
    }
  }
  return any;
}

// Raw values of one row for this lane (prefetch ring) ...
struct Raw {
  float r, q, p, h, x;
  uint32_t m;   // imask
  int32_t lab;  // label (mixed items only)
};

// ... and a row of the compute ring: r_k and p_k = r_k + beta p_{k-1}
// formed with the pixel's own component (only intra-component neighbours
// are ever read, and those share the centre's alpha and beta).
struct Row {
  float rn, pn, h, xn;
  uint32_t m;  // imask | (slot + 1) << 8
};

template <bool PURE>
__device__ __forceinline__ Raw load_raw(const FillArgs& a, int par, int y, int ylim, int x) {
  Raw w;
  w.r = w.q = w.p = w.h = w.x = 0.f;
  w.m = 0;
  w.lab = -1;
  if (y >= 0 && y <= ylim && x >= 0 && x < a.W) {
    const int64_t i = int64_t(y) * a.W + x;
    w.r = __ldcg(a.r[par] + i);
    w.q = __ldcg(a.q[par] + i);
    w.p = __ldcg(a.p[par] + i);
    w.x = __ldcg(a.x + i);
    w.h = __ldg(a.hw + i);
    w.m = __ldg(a.imask + i);
    if (!PURE) w.lab = __ldg(a.labels + i);
  }
  return w;
}

template <bool PURE>
__device__ __forceinline__ Row to_row(const Raw& w, const Item& it, const Coefs& k) {
  Row o;
  float al = k.al[0], be = k.be[0];
  uint32_t m = w.m;
  if (!PURE) {
    const int s = slot_of(it, w.lab);
    al = 0.f;
    be = 0.f;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
      if (j == s) {
        al = k.al[j];
        be = k.be[j];
      }
    m |= uint32_t(s + 1) << 8;
  } else {
    m |= 1u << 8;
  }
  o.rn = fmaf(-al, w.q, w.r);
  o.pn = fmaf(be, w.p, o.rn);
  o.xn = fmaf(al, w.p, w.x);
  o.h = w.h;
  o.m = m;
  return o;
}

// One CG sweep over one item (see the header).
template <int CONN, bool PURE>
__device__ __forceinline__ void sweep_item(const FillArgs& a, const Item& it, int par) {
  const int lane = threadIdx.x & 31;
  Coefs k;
  if (!item_coefs(a, it, k)) return;
  const int x = it.x0 - 1 + lane;
  const bool center_lane = lane >= 1 && lane <= SW && x < a.W;
  float* rout = a.r[par ^ 1];
  float* qout = a.q[par ^ 1];
  float* pout = a.p[par ^ 1];
  double acc[SLOTS][NDOT];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
#pragma unroll
    for (int d = 0; d < NDOT; ++d) acc[j][d] = 0.0;
  const int yend = min(it.y0 + SH, a.rows);
  const int ylim = min(yend, a.rows - 1);  // last row the stencil touches
  Raw F[PF];
#pragma unroll
  for (int t = 0; t < PF; ++t) F[t] = load_raw<PURE>(a, par, it.y0 + 2 + t, ylim, x);
  Row U = to_row<PURE>(load_raw<PURE>(a, par, it.y0 - 1, ylim, x), it, k);
  Row C = to_row<PURE>(load_raw<PURE>(a, par, it.y0, ylim, x), it, k);
  Row D = to_row<PURE>(load_raw<PURE>(a, par, it.y0 + 1, ylim, x), it, k);
  for (int y = it.y0; y < yend; ++y) {
    const Raw N = load_raw<PURE>(a, par, y + 2 + PF, ylim, x);  // PF rows in flight
    const int s = PURE ? 0 : int(C.m >> 8) - 1;  // this pixel's slot, -1: not in the item
    uint8_t st = ST_IDLE;
    if (PURE) {
      st = k.st[0];
    } else {
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        if (j == s) st = k.st[j];
    }
    const bool on = center_lane && (C.m & 0xFF) != 0;
    const float pa = C.pn;
    const float ha = C.h;
    const uint32_t m = C.m;
    float q = 0.f;
#define NI_NB(pp, hh) fmaf(ha + (hh), pa - (pp), q)
#define NI_UP(v) __shfl_up_sync(0xffffffffu, (v), 1)
#define NI_DN(v) __shfl_down_sync(0xffffffffu, (v), 1)
    {
      const float pCl = NI_UP(C.pn), hCl = NI_UP(C.h);
      const float pCr = NI_DN(C.pn), hCr = NI_DN(C.h);
      if (CONN == 8) {
        const float pDl = NI_UP(D.pn), hDl = NI_UP(D.h);
        const float pDr = NI_DN(D.pn), hDr = NI_DN(D.h);
        const float pUl = NI_UP(U.pn), hUl = NI_UP(U.h);
        const float pUr = NI_DN(U.pn), hUr = NI_DN(U.h);
        if (m & 0x01) q = NI_NB(pCr, hCr);    // (+1, 0)
        if (m & 0x02) q = NI_NB(pDl, hDl);    // (-1,+1)
        if (m & 0x04) q = NI_NB(D.pn, D.h);   // ( 0,+1)
        if (m & 0x08) q = NI_NB(pDr, hDr);    // (+1,+1)
        if (m & 0x10) q = NI_NB(pCl, hCl);    // (-1, 0)
        if (m & 0x20) q = NI_NB(pUr, hUr);    // (+1,-1)
        if (m & 0x40) q = NI_NB(U.pn, U.h);   // ( 0,-1)
        if (m & 0x80) q = NI_NB(pUl, hUl);    // (-1,-1)
      } else {
        if (m & 0x01) q = NI_NB(pCr, hCr);    // (+1, 0)
        if (m & 0x02) q = NI_NB(D.pn, D.h);   // ( 0,+1)
        if (m & 0x10) q = NI_NB(pCl, hCl);    // (-1, 0)
        if (m & 0x20) q = NI_NB(U.pn, U.h);   // ( 0,-1)
      }
    }
#undef NI_NB
#undef NI_UP
#undef NI_DN
    if (on && st == ST_ACTIVE) {
      const int64_t i = int64_t(y) * a.W + x;
      __stcg(rout + i, C.rn);
      __stcg(pout + i, pa);
      __stcg(qout + i, q);
      __stcg(a.x + i, C.xn);
      const double dp = pa, dq = q, dr = C.rn;
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        if (j == s) {
          acc[j][0] = fma(dp, dq, acc[j][0]);
          acc[j][1] = fma(dr, dq, acc[j][1]);
          acc[j][2] = fma(dq, dq, acc[j][2]);
          acc[j][3] = fma(dr, dr, acc[j][3]);
        }
    } else if (on && st == ST_FLUSH) {
      __stcg(a.x + int64_t(y) * a.W + x, C.xn);  // the pending x_{k+1}
    }
    U = C;
    C = D;
    D = to_row<PURE>(F[0], it, k);
#pragma unroll
    for (int t = 0; t < PF - 1; ++t) F[t] = F[t + 1];
    F[PF - 1] = N;
  }
  bool live[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) live[j] = k.st[j] == ST_ACTIVE || k.st[j] == ST_FLUSH;
  item_finish(a, it, acc, live, [&](int32_t c, const double* d) {
    if (__ldcg(a.status + c) == ST_FLUSH) {  // the pending update is applied
      a.status[c] = __ldcg(a.final_status + c);
      atomicSub(a.active, 1);
      atomicExch(a.changed, 1);
      return;
    }
    const double pq = d[0], rq = d[1], qq = d[2], rr = d[3];
    const int n = __ldcg(a.iters + c) + 1;  // updates once this sweep's alpha is applied
    a.iters[c] = n;
    a.rho[c] = rr;
    double alpha = 0.0, rho1 = 0.0;
    bool stop = false;
    uint8_t fin = ST_CONVERGED;
    if (pq > 0.0) {
      alpha = rr / pq;
      rho1 = rr - 2.0 * alpha * rq + alpha * alpha * qq;
      if (rho1 < 0.0) rho1 = 0.0;
      if (n < __ldcg(a.cap + c) && sqrt(rho1) < __ldcg(a.tol + c)) {
        stop = true;  // scipy's top-of-loop test before iteration n
      } else if (n >= __ldcg(a.cap + c)) {
        stop = true;  // loop exhausted: info = maxiter
        fin = ST_CAPPED;
      }
    } else {
      stop = true;  // breakdown: p in the null space (only once r == 0)
    }
    a.alpha[c] = alpha;
    if (stop) {
      a.final_status[c] = fin;
      a.status[c] = ST_FLUSH;
      atomicExch(a.changed, 1);
    } else {
      a.beta[c] = rho1 / rr;
      a.rho[c] = rho1;
    }
  });
}

// Rebuild the list of items with an ACTIVE or FLUSH component (order is
// irrelevant: the partial slots are fixed per item).
__device__ void rebuild_items(const FillArgs& a, int dst, int gwarp, int nwarps) {
  const int lane = threadIdx.x & 31;
  for (int k0 = gwarp * 32; k0 < a.nitems; k0 += nwarps * 32) {
    const int k = k0 + lane;
    bool act = false;
    if (k < a.nitems) {
      const Item it = a.items[k];
      const int n = item_n(it);
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        if (j < n) {
          const uint8_t st = __ldcg(a.status + it.comp[j]);
          if (st == ST_ACTIVE || st == ST_FLUSH) act = true;
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, act);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(a.nactive_items + dst, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (act) a.active_items[dst * a.nitems + base + __popc(m & ((1u << lane) - 1))] = k;
  }
}

template <int CONN, int MINB>
__global__ void __launch_bounds__(NT, MINB) fill_cg_kernel(FillArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int gwarp = blockIdx.x * WPB + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * WPB;
  int cur = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.nactive_items[0] = 0;
    a.nactive_items[1] = 0;
  }
  grid.sync();
  rebuild_items(a, 0, gwarp, nwarps);
  grid.sync();
  for (int it = 0;; ++it) {
    if (__ldcg(a.active) == 0) break;
    const int par = it & 1;
    const int n = __ldcg(a.nactive_items + cur);
    for (int k = gwarp; k < n; k += nwarps) {
      const Item item = a.items[__ldcg(a.active_items + cur * a.nitems + k)];
      if (item_pure(item)) sweep_item<CONN, true>(a, item, par);
      else sweep_item<CONN, false>(a, item, par);
    }
    grid.sync();
    if (__ldcg(a.changed)) {
      const int nxt = cur ^ 1;
      if (blockIdx.x == 0 && threadIdx.x == 0) a.nactive_items[nxt] = 0;
      grid.sync();
      rebuild_items(a, nxt, gwarp, nwarps);
      grid.sync();
      if (blockIdx.x == 0 && threadIdx.x == 0) *a.changed = 0;
      cur = nxt;
      grid.sync();
    }
  }
}

// Initial ||b||^2 per component and the state of every component.  One warp
// per item, like the sweeps.
__global__ void __launch_bounds__(NT) init_norm_kernel(FillArgs a, double rtol) {
  const int gwarp = blockIdx.x * WPB + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * WPB;
  const int lane = threadIdx.x & 31;
  for (int k = gwarp; k < a.nitems; k += nwarps) {
    const Item it = a.items[k];
    const int x = it.x0 - 1 + lane;
    const bool on = lane >= 1 && lane <= SW && x < a.W;
    double acc[SLOTS][NDOT];
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
#pragma unroll
      for (int d = 0; d < NDOT; ++d) acc[j][d] = 0.0;
    const int yend = min(it.y0 + SH, a.rows);
    if (on) {
      for (int y = it.y0; y < yend; ++y) {
        const int64_t i = int64_t(y) * a.W + x;
        const int s = slot_of(it, a.labels[i]);
        if (s < 0) continue;
        const double rv = a.r[0][i];
#pragma unroll
        for (int j = 0; j < SLOTS; ++j)
          if (j == s) acc[j][3] += rv * rv;
      }
    }
    bool live[SLOTS] = {true, true};
    item_finish(a, it, acc, live, [&](int32_t c, const double* d) {
      const double bb = d[3];
      a.rho[c] = bb;
      const double bn = sqrt(bb);
      a.tol[c] = rtol * bn;
      a.iters[c] = 0;
      a.alpha[c] = 0.0;
      a.beta[c] = 0.0;
      // scipy: bnrm2 == 0 -> x = 0; then the first top-of-loop test
      if (bb == 0.0 || bn < rtol * bn) {
        a.status[c] = ST_CONVERGED;
      } else if (a.cap[c] <= 0) {
        a.status[c] = ST_CAPPED;
      } else {
        a.status[c] = ST_ACTIVE;
        atomicAdd(a.active, 1);
      }
    });
  }
}

// status ACTIVE only while the initial norm pass counts arrivals; its
// finaliser sets the real state and the active count.
__global__ void init_state_kernel(FillArgs a, const int32_t* __restrict__ comp_size, int C,
                                  int cg_max_iters) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    a.status[c] = comp_size[c] >= 2 ? ST_ACTIVE : ST_IDLE;
    a.final_status[c] = ST_CONVERGED;
    a.iters[c] = 0;
    const int n = comp_size[c];
    a.cap[c] = n > cg_max_iters ? n : cg_max_iters;
    a.rho[c] = 0.0;
  }
}

__global__ void output_kernel(const float* __restrict__ x, const int32_t* __restrict__ labels,
                              const int32_t* __restrict__ comp_size, int64_t npix,
                              double* __restrict__ z) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t l = labels[i];
    z[i] = (l >= 0 && comp_size[l] >= 2) ? double(x[i]) : 0.0;
  }
}

__global__ void status_out_kernel(const FillArgs a, int C, const int32_t* __restrict__ comp_size,
                                  int32_t* __restrict__ iters_out,
                                  int32_t* __restrict__ status_out,
                                  unsigned long long* __restrict__ px_iters,
                                  int32_t* __restrict__ max_iters) {
  unsigned long long acc = 0;
  int mx = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int it = a.iters[c];
    iters_out[c] = it;
    status_out[c] = a.status[c] == ST_CAPPED ? 1 : 0;
    if (comp_size[c] >= 2) acc += (unsigned long long)comp_size[c] * (unsigned long long)it;
    mx = it > mx ? it : mx;
  }
  atomicAdd(px_iters, acc);
  atomicMax(max_iters, mx);
}

// ------------------------------------------------------------ workspace

struct FillWs {
  float *x, *r0, *r1, *q0, *q1, *p0, *p1, *hw;
  uint8_t* imask;
  int32_t *slot_base, *nslots, *nitems_strip, *item_base, *strip_comps, *partial_comp,
      *partial_idx, *plist, *keys_sorted;
  Item* items;
  int32_t *comp_size, *comp_nparts, *comp_pstart, *comp_cnt, *iters, *cap, *active, *changed,
      *total, *total_items, *active_items, *nactive_items;
  double *partial, *rho, *alpha, *beta, *tol;
  uint8_t *status, *final_status;
  unsigned long long* px_iters;
  int32_t* max_iters;
  void* sort_ws;
  size_t sort_bytes;
  void* scan_ws;
};

static void carve_fill(Carver& c, FillWs& w, int64_t npix, int nstrips, int C) {
  // every partial slot owns >= 1 pixel
  const int64_t P = npix;
  const int64_t NI = nstrips + P / SLOTS + 1;  // items
  w.x = c.take<float>(npix);
  w.r0 = c.take<float>(npix);
  w.r1 = c.take<float>(npix);
  w.q0 = c.take<float>(npix);
  w.q1 = c.take<float>(npix);
  w.p0 = c.take<float>(npix);
  w.p1 = c.take<float>(npix);
  w.hw = c.take<float>(npix);
  w.imask = c.take<uint8_t>(npix);
  w.slot_base = c.take<int32_t>(nstrips + 1);
  w.nslots = c.take<int32_t>(nstrips + 1);
  w.nitems_strip = c.take<int32_t>(nstrips + 1);
  w.item_base = c.take<int32_t>(nstrips + 1);
  w.strip_comps = c.take<int32_t>(int64_t(nstrips) * SPX);
  w.items = c.take<Item>(NI);
  w.active_items = c.take<int32_t>(2 * NI);
  w.nactive_items = c.take<int32_t>(2);
  w.partial_comp = c.take<int32_t>(P);
  w.partial_idx = c.take<int32_t>(P);
  w.plist = c.take<int32_t>(P);
  w.keys_sorted = c.take<int32_t>(P);
  w.partial = c.take<double>(P * NDOT);
  w.comp_size = c.take<int32_t>(C + 1);
  w.comp_nparts = c.take<int32_t>(C + 1);
  w.comp_pstart = c.take<int32_t>(C + 1);
  w.comp_cnt = c.take<int32_t>(C + 1);
  w.iters = c.take<int32_t>(C + 1);
  w.cap = c.take<int32_t>(C + 1);
  w.rho = c.take<double>(C + 1);
  w.alpha = c.take<double>(C + 1);
  w.beta = c.take<double>(C + 1);
  w.tol = c.take<double>(C + 1);
  w.status = c.take<uint8_t>(C + 1);
  w.final_status = c.take<uint8_t>(C + 1);
  w.active = c.take<int32_t>(1);
  w.changed = c.take<int32_t>(1);
  w.total = c.take<int32_t>(1);
  w.total_items = c.take<int32_t>(1);
  w.px_iters = c.take<unsigned long long>(1);
  w.max_iters = c.take<int32_t>(1);
  w.sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, w.sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)P);
  w.sort_ws = c.take<char>(w.sort_bytes);
  const int64_t scan_n = (nstrips + 1) > (C + 1) ? (nstrips + 1) : (C + 1);
  w.scan_ws = c.take<char>(scan_ws_bytes(scan_n));
}

}  // namespace ni

using namespace ni;

static void strip_grid(int B, int H, int W, int* nsx, int* nsy) {
  *nsx = div_up(W, SW);
  *nsy = div_up(int64_t(B) * H, SH);
}

extern "C" int ni_fill_workspace_size(int B, int H, int W, int connectivity, int count,
                                      size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  const int64_t npix = int64_t(B) * H * W;
  int nsx, nsy;
  strip_grid(B, H, W, &nsx, &nsy);
  Sizer s;
  FillWs w;
  carve_fill(s, w, npix, nsx * nsy, count);
  *bytes = s.used;
  return NI_OK;
}

extern "C" int ni_fill(const int32_t* labels, int count, const double* omega_a,
                       const double* omega_b, const double* gamma, const uint8_t* eflags, int B,
                       int H, int W, int connectivity, int model, double cg_tol, int cg_max_iters,
                       double* z_out, int32_t* comp_iters, int32_t* comp_status, void* workspace,
                       size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(model == 0 || (model == 1 && connectivity == 4), "bad model/connectivity");
  NI_CHECK_ARG(cg_tol > 0, "cg_tol must be positive");
  NI_CHECK_ARG(count >= 0, "count must be non-negative");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  const int rows = B * H;
  int nsx, nsy;
  strip_grid(B, H, W, &nsx, &nsy);
  const int nstrips = nsx * nsy;
  Carver cv(workspace, workspace_bytes);
  FillWs w;
  carve_fill(cv, w, npix, nstrips, count);
  if (!cv.ok() || !workspace) {
    set_error("ni_fill: workspace too small (%zu < %zu)", workspace_bytes, cv.used);
    return NI_ERR_WORKSPACE;
  }
  const int blocks = int(std::min<int64_t>((npix + 255) / 256, int64_t(kSMs) * 16));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_size, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_nparts, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_cnt, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.active, 0, sizeof(int32_t), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.changed, 0, sizeof(int32_t), s));
#define NI_PREP(CONN, MODEL)                                                                   \
  NI_COUNT_LAUNCH(), prep_kernel<CONN, MODEL><<<blocks, 256, 0, s>>>(                          \
                         labels, omega_a, omega_b, gamma, eflags, H, W, npix, w.hw, w.imask,   \
                         w.x, w.r0, w.r1, w.q0, w.q1, w.p0, w.p1, w.comp_size)
  if (connectivity == 8) NI_PREP(8, 0);
  else if (model == 0) NI_PREP(4, 0);
  else NI_PREP(4, 1);
#undef NI_PREP
  NI_LAUNCH_CHECK();
  // ---- static reduction plan: strips -> items -> partial slots
  NI_COUNT_LAUNCH(), strip_comps_kernel<<<nstrips, NT, 0, s>>>(labels, w.comp_size, rows, W, nsx,
                                                              w.nslots, w.strip_comps);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(w.nslots, w.slot_base, nstrips, w.total, w.scan_ws, s));
  NI_COUNT_LAUNCH(), item_counts_kernel<<<div_up(nstrips, 256), 256, 0, s>>>(w.nslots, nstrips,
                                                                            w.nitems_strip);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(w.nitems_strip, w.item_base, nstrips, w.total_items, w.scan_ws, s));
  NI_COUNT_LAUNCH(), strip_items_kernel<<<div_up(nstrips, 128), 128, 0, s>>>(
                         w.nslots, w.slot_base, w.item_base, w.strip_comps, nstrips, nsx, w.items,
                         w.partial_comp, w.partial_idx, w.comp_nparts);
  NI_LAUNCH_CHECK();
  int32_t P = 0, NIt = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&P, w.total, sizeof(P), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaMemcpyAsync(&NIt, w.total_items, sizeof(NIt), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  if (P > 0) {
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= count) ++end_bit;
    size_t sb = w.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_ws, sb, w.partial_comp, w.keys_sorted,
                                                w.partial_idx, w.plist, P, 0, end_bit, s));
  }
  NI_TRY(exclusive_scan_i32(w.comp_nparts, w.comp_pstart, count + 1, nullptr, w.scan_ws, s));
  FillArgs a;
  a.rows = rows;
  a.W = W;
  a.x = w.x;
  a.r[0] = w.r0;
  a.r[1] = w.r1;
  a.q[0] = w.q0;
  a.q[1] = w.q1;
  a.p[0] = w.p0;
  a.p[1] = w.p1;
  a.hw = w.hw;
  a.imask = w.imask;
  a.labels = labels;
  a.items = w.items;
  a.nitems = NIt;
  a.comp_pstart = w.comp_pstart;
  a.comp_plist = w.plist;
  a.comp_cnt = w.comp_cnt;
  a.partial = w.partial;
  a.active_items = w.active_items;
  a.nactive_items = w.nactive_items;
  a.rho = w.rho;
  a.alpha = w.alpha;
  a.beta = w.beta;
  a.tol = w.tol;
  a.iters = w.iters;
  a.cap = w.cap;
  a.status = w.status;
  a.final_status = w.final_status;
  a.active = w.active;
  a.changed = w.changed;
  if (count > 0) {
    NI_COUNT_LAUNCH(), init_state_kernel<<<div_up(count, 256), 256, 0, s>>>(a, w.comp_size, count,
                                                                           cg_max_iters);
    NI_LAUNCH_CHECK();
  }
  if (NIt > 0) {
    NI_COUNT_LAUNCH(), init_norm_kernel<<<div_up(NIt, WPB), NT, 0, s>>>(a, cg_tol);
    NI_LAUNCH_CHECK();
  }
  // ---- the whole CG: one persistent cooperative launch
  {
    // occupancy variant (experiments): NI_FILL_MINB = CTAs/SM the register
    // budget is sized for (2: 128 regs, 3: 80, 4: 64)
    const char* mb = getenv("NI_FILL_MINB");
    const int minb = mb ? atoi(mb) : 3;
    void* kfn;
    if (connectivity == 8)
      kfn = minb == 2 ? (void*)fill_cg_kernel<8, 2>
                      : (minb == 4 ? (void*)fill_cg_kernel<8, 4> : (void*)fill_cg_kernel<8, 3>);
    else
      kfn = minb == 2 ? (void*)fill_cg_kernel<4, 2>
                      : (minb == 4 ? (void*)fill_cg_kernel<4, 4> : (void*)fill_cg_kernel<4, 3>);
    int dev = 0, sms = 0, per_sm = 0;
    NI_CUDA_TRY(cudaGetDevice(&dev));
    NI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    NI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NT, 0));
    int G = per_sm * sms;
    const int need = div_up(NIt > 0 ? NIt : 1, WPB);
    if (G > need) G = need;
    if (G < 1) G = 1;
    void* args[] = {&a};
    cudaEvent_t e0, e1;
    NI_CUDA_TRY(cudaEventCreate(&e0));
    NI_CUDA_TRY(cudaEventCreate(&e1));
    NI_CUDA_TRY(cudaEventRecord(e0, s));
    NI_COUNT_LAUNCH();
    NI_CUDA_TRY(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(NT), args, 0, s));
    NI_CUDA_TRY(cudaEventRecord(e1, s));
    g_fill_report.grid = G;
    g_fill_report.ntiles = NIt;
    g_fill_report.npartials = P;
    NI_CUDA_TRY(cudaMemsetAsync(w.px_iters, 0, sizeof(unsigned long long), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.max_iters, 0, sizeof(int32_t), s));
    if (count > 0) {
      NI_COUNT_LAUNCH(), status_out_kernel<<<div_up(count, 256), 256, 0, s>>>(
                             a, count, w.comp_size, comp_iters, comp_status, w.px_iters,
                             w.max_iters);
      NI_LAUNCH_CHECK();
    }
    NI_COUNT_LAUNCH(), output_kernel<<<blocks, 256, 0, s>>>(w.x, labels, w.comp_size, npix, z_out);
    NI_LAUNCH_CHECK();
    unsigned long long pxi = 0;
    int32_t mxi = 0;
    NI_CUDA_TRY(cudaMemcpyAsync(&pxi, w.px_iters, sizeof(pxi), cudaMemcpyDeviceToHost, s));
    NI_CUDA_TRY(cudaMemcpyAsync(&mxi, w.max_iters, sizeof(mxi), cudaMemcpyDeviceToHost, s));
    NI_CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    NI_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    g_fill_report.cg_ms = ms;
    g_fill_report.px_iters = (long long)pxi;
    g_fill_report.max_iters = mxi;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return NI_OK;
}

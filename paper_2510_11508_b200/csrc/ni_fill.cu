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
//   x, r, q, p[2] : float32 CG vectors (p double-buffered: sweep 1 reads the
//                   neighbours' previous p while other warps write the new)
//   hw            : float32 W_a = gamma_a^2 / 2  (c_ab = hw_a + hw_b)
//   imask         : uint8, bit k = forward edge k intra-component and valid,
//                   bit 4+k = backward edge k (pixel - offset_k)
//
// Work decomposition: the grid is cut into strips of 30 columns x 32 rows.
// A warp processes a strip by marching down its rows with a register ring
// of rows y-1, y, y+1 (+ prefetched rows); lanes 0 and 31 carry the left /
// right halo columns, so horizontal neighbours are warp shuffles and there
// is no block barrier anywhere in a sweep.  A strip touching several
// multi-pixel components becomes ceil(n/4) "items" of <= 4 components that
// read the int32 labels; a strip with one component (the common case) is a
// "pure" item that needs no label at all (singletons / invalid pixels carry
// r = p = 0 and stay 0 under any update).
//
// Reductions are deterministic: each item writes one float64 partial per
// component (lane-local sums over rows, fixed xor tree over lanes); the last
// warp to arrive for a component (integer counter) sums the component's
// partials in plan order and updates its scalars.  Two grid syncs per
// iteration:
//   sweep 1: p' = r + beta p ; q = A p' ; <p', q>   -> alpha
//   sweep 2: x += alpha p' ; r -= alpha q ; <r, r>  -> stop test, beta
// Algorithmic bytes per active pixel and iteration (pure items):
//   sweep 1: read r, p, hw, imask (13 B), write p', q (8 B)
//   sweep 2: read x, r, p', q (16 B), write x, r (8 B)          => 45 B/px
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
constexpr int SLOTS = 4;  // components per item
constexpr int PF = 4;     // rows prefetched ahead in sweep 1

enum : uint8_t { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_CAPPED = 2, ST_IDLE = 3 };

// One work item: a strip and up to 4 of its components.
struct __align__(16) Item {
  int32_t x0, y0;  // top-left pixel of the strip (column of lane 1)
  int32_t pbase;   // first partial slot of this item
  int32_t flags;   // bits 0-7: components in the item (1..4); bit 8: pure strip
  int32_t comp[SLOTS];
};

__device__ __forceinline__ int item_n(const Item& it) { return it.flags & 0xFF; }
__device__ __forceinline__ bool item_pure(const Item& it) { return (it.flags >> 8) & 1; }

struct FillArgs {
  int rows, W;
  float* x;
  float* r;
  float* q;
  float* p0;
  float* p1;
  const float* hw;
  const uint8_t* imask;
  const int32_t* labels;
  // plan
  const Item* items;
  int nitems;
  const int32_t* comp_pstart;  // [C+1] partial range per component
  const int32_t* comp_plist;   // [P] partial indices grouped by component
  int32_t* comp_cnt;           // [C] arrival counters (zero between sweeps)
  double* partial;             // [P]
  int32_t* active_items;       // [2][nitems]
  int32_t* nactive_items;      // [2]
  // component state
  double* rho;
  double* alpha;
  double* beta;
  double* tol;
  int32_t* iters;
  int32_t* cap;
  uint8_t* status;
  uint8_t* brk;      // breakdown flag set in sweep 1, resolved in sweep 2
  int32_t* active;   // number of active components
  int32_t* changed;  // a component finished during the last sweep 2
};

// ----------------------------------------------------------------- setup

template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) prep_kernel(
    const int32_t* __restrict__ labels, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int64_t npix, float* __restrict__ hw,
    uint8_t* __restrict__ imask, float* __restrict__ x, float* __restrict__ r,
    float* __restrict__ p0, float* __restrict__ p1, float* __restrict__ q,
    int32_t* __restrict__ comp_size) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t lab = labels[i];
    x[i] = 0.f;
    p0[i] = 0.f;
    p1[i] = 0.f;
    q[i] = 0.f;
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

// Write the item's per-component partials, count arrivals, and let the last
// arriving warp of a component reduce its partials in plan order.
template <class Fin>
__device__ __forceinline__ void item_finish(const FillArgs& a, const Item& it, const double* acc,
                                            Fin fin) {
  const int lane = threadIdx.x & 31;
  const int n = item_n(it);
  double tot[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) tot[s] = warp_sum(acc[s]);
  unsigned last = 0;
  if (lane < n) {
    double v = tot[0];
    int32_t c = it.comp[0];
#pragma unroll
    for (int s = 1; s < SLOTS; ++s)
      if (lane == s) {
        v = tot[s];
        c = it.comp[s];
      }
    if (__ldcg(a.status + c) == ST_ACTIVE) {
      a.partial[it.pbase + lane] = v;
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
    double sum = 0.0;
    for (int j = q0 + lane; j < q1; j += 32) sum += __ldcg(a.partial + a.comp_plist[j]);
    sum = warp_sum(sum);
    if (lane == 0) {
      fin(c, sum);
      a.comp_cnt[c] = 0;
    }
    __syncwarp();
  }
}

__device__ __forceinline__ int slot_of(const Item& it, int32_t lab) {
  int s = -1;
  const int n = item_n(it);
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
    if (j < n && it.comp[j] == lab) s = j;
  return s;
}

// Item coefficients for one sweep: value (beta or alpha) and activity.
__device__ __forceinline__ bool item_coefs(const FillArgs& a, const Item& it, int which,
                                           float* coef, bool* act) {
  bool any = false;
  const int n = item_n(it);
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) {
    coef[j] = 0.f;
    act[j] = false;
    if (j < n) {
      const int32_t c = it.comp[j];
      act[j] = __ldcg(a.status + c) == ST_ACTIVE;
      coef[j] = float(which == 0 ? __ldcg(a.beta + c) : __ldcg(a.alpha + c));
      any |= act[j];
    }
  }
  return any;
}

// Raw values of one row for this lane (prefetch ring) ...
struct Raw {
  float r, p, h;
  uint32_t m;    // imask
  int32_t lab;   // label (mixed items only)
};

// ... and a row of the compute ring, with p' = r + beta p already formed
// using the pixel's own component (only intra-component neighbours are ever
// read, and those share the centre's component and beta).
struct Row {
  float pn, h;
  uint32_t m;  // imask | (slot + 1) << 8  (slot 0 for pure items)
};

__device__ __forceinline__ Raw load_raw(const FillArgs& a, const float* __restrict__ pin, int y,
                                        int ylim, int x, bool pure) {
  Raw w;
  w.r = w.p = w.h = 0.f;
  w.m = 0;
  w.lab = -1;
  if (y >= 0 && y <= ylim && x >= 0 && x < a.W) {
    const int64_t i = int64_t(y) * a.W + x;
    w.r = __ldcg(a.r + i);
    w.p = __ldcg(pin + i);
    w.h = __ldg(a.hw + i);
    w.m = __ldg(a.imask + i);
    if (!pure) w.lab = __ldg(a.labels + i);
  }
  return w;
}

__device__ __forceinline__ Row to_row(const Raw& w, const Item& it, const float* beta) {
  Row o;
  float b = beta[0];
  uint32_t m = w.m;
  if (!item_pure(it)) {
    const int s = slot_of(it, w.lab);
    b = 0.f;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
      if (j == s) b = beta[j];
    m |= uint32_t(s + 1) << 8;
  } else {
    m |= 1u << 8;
  }
  o.pn = fmaf(b, w.p, w.r);
  o.h = w.h;
  o.m = m;
  return o;
}

// sweep 1 over one item
template <int CONN>
__device__ __forceinline__ void sweep1_item(const FillArgs& a, const Item& it,
                                            const float* __restrict__ pin,
                                            float* __restrict__ pout) {
  const int lane = threadIdx.x & 31;
  float beta[SLOTS];
  bool act[SLOTS];
  if (!item_coefs(a, it, 0, beta, act)) return;
  const bool pure = item_pure(it);
  const int x = it.x0 - 1 + lane;
  const bool center_lane = lane >= 1 && lane <= SW && x < a.W;
  double acc[SLOTS] = {0.0, 0.0, 0.0, 0.0};
  // compute ring U = y-1, C = y, D = y+1; raw prefetch ring F = y+2 .. y+1+PF
  const int yend = min(it.y0 + SH, a.rows);
  const int ylim = min(yend, a.rows - 1);  // last row the stencil touches
  Raw F[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) F[k] = load_raw(a, pin, it.y0 + 2 + k, ylim, x, pure);
  Row U = to_row(load_raw(a, pin, it.y0 - 1, ylim, x, pure), it, beta);
  Row C = to_row(load_raw(a, pin, it.y0, ylim, x, pure), it, beta);
  Row D = to_row(load_raw(a, pin, it.y0 + 1, ylim, x, pure), it, beta);
  for (int y = it.y0; y < yend; ++y) {
    const Raw N = load_raw(a, pin, y + 2 + PF, ylim, x, pure);  // PF rows in flight
    const int s = int(C.m >> 8) - 1;  // this pixel's slot, -1: not in the item
    bool mine = center_lane && (C.m & 0xFF) != 0 && s >= 0;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
      if (j == s) mine = mine && act[j];
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
    if (mine) {
      const int64_t i = int64_t(y) * a.W + x;
      __stcg(pout + i, pa);
      __stcg(a.q + i, q);
      const double v = double(pa) * double(q);
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        if (j == s) acc[j] += v;
    }
    U = C;
    C = D;
    D = to_row(F[0], it, beta);
#pragma unroll
    for (int k = 0; k < PF - 1; ++k) F[k] = F[k + 1];
    F[PF - 1] = N;
  }
  item_finish(a, it, acc, [&](int32_t c, double pq) {
    if (pq > 0.0) {
      a.alpha[c] = __ldcg(a.rho + c) / pq;
    } else {  // breakdown (p' in the null space): resolved in sweep 2
      a.alpha[c] = 0.0;
      a.brk[c] = 1;
    }
  });
}

// sweep 2 over one item.  Pixels without intra edges (and singletons /
// invalid pixels) have p' = q = 0, so x and r are unchanged there: pure items
// need neither imask nor labels, and the stores are skipped.
constexpr int U2 = 4;  // rows per batch of loads
__device__ __forceinline__ void sweep2_item(const FillArgs& a, const Item& it,
                                            const float* __restrict__ pnew) {
  const int lane = threadIdx.x & 31;
  float alpha[SLOTS];
  bool act[SLOTS];
  if (!item_coefs(a, it, 1, alpha, act)) return;
  const bool pure = item_pure(it);
  const int x = it.x0 - 1 + lane;
  const bool on = lane >= 1 && lane <= SW && x < a.W;
  double acc[SLOTS] = {0.0, 0.0, 0.0, 0.0};
  const int yend = min(it.y0 + SH, a.rows);
  for (int y0 = it.y0; y0 < yend; y0 += U2) {
    float xv[U2], rv[U2], pv[U2], qv[U2];
    int32_t lab[U2];
#pragma unroll
    for (int k = 0; k < U2; ++k) {
      const int y = y0 + k;
      xv[k] = rv[k] = pv[k] = qv[k] = 0.f;
      lab[k] = -1;
      if (on && y < yend) {
        const int64_t i = int64_t(y) * a.W + x;
        pv[k] = __ldcg(pnew + i);
        qv[k] = __ldcg(a.q + i);
        rv[k] = __ldcg(a.r + i);
        xv[k] = __ldcg(a.x + i);
        if (!pure) lab[k] = __ldg(a.labels + i);
      }
    }
#pragma unroll
    for (int k = 0; k < U2; ++k) {
      const int y = y0 + k;
      int s = 0;
      float al = alpha[0];
      bool mine = on && y < yend && act[0];
      if (!pure) {
        s = slot_of(it, lab[k]);
        mine = on && y < yend && s >= 0;
#pragma unroll
        for (int j = 0; j < SLOTS; ++j)
          if (j == s) {
            al = alpha[j];
            mine = mine && act[j];
          }
      }
      if (!mine) continue;
      const int64_t i = int64_t(y) * a.W + x;
      if (pv[k] != 0.f) __stcg(a.x + i, fmaf(al, pv[k], xv[k]));
      const float rn = fmaf(-al, qv[k], rv[k]);
      if (qv[k] != 0.f) __stcg(a.r + i, rn);
      const double v = double(rn) * double(rn);
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        if (j == s) acc[j] += v;
    }
  }
  item_finish(a, it, acc, [&](int32_t c, double rr) {
    const int itn = __ldcg(a.iters + c) + 1;
    a.iters[c] = itn;
    bool done = false;
    if (__ldcg(a.brk + c)) {
      a.status[c] = ST_CONVERGED;
      done = true;
    } else if (itn < __ldcg(a.cap + c) && sqrt(rr) < __ldcg(a.tol + c)) {  // scipy's top-of-loop test
      a.status[c] = ST_CONVERGED;
      done = true;
    } else if (itn >= __ldcg(a.cap + c)) {  // loop exhausted: info = maxiter
      a.status[c] = ST_CAPPED;
      done = true;
    } else {
      a.beta[c] = rr / __ldcg(a.rho + c);
      a.rho[c] = rr;
    }
    if (done) {
      atomicSub(a.active, 1);
      atomicExch(a.changed, 1);
    }
  });
}

// Rebuild the list of items with an active component (order irrelevant: the
// partial slots are fixed per item).
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
        if (j < n && __ldcg(a.status + it.comp[j]) == ST_ACTIVE) act = true;
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
    const float* pin = (it & 1) ? a.p1 : a.p0;
    float* pout = (it & 1) ? a.p0 : a.p1;
    const int n = __ldcg(a.nactive_items + cur);
    for (int k = gwarp; k < n; k += nwarps) {
      const Item item = a.items[__ldcg(a.active_items + cur * a.nitems + k)];
      sweep1_item<CONN>(a, item, pin, pout);
    }
    grid.sync();
    for (int k = gwarp; k < n; k += nwarps) {
      const Item item = a.items[__ldcg(a.active_items + cur * a.nitems + k)];
      sweep2_item(a, item, pout);
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
    double acc[SLOTS] = {0.0, 0.0, 0.0, 0.0};
    const int yend = min(it.y0 + SH, a.rows);
    if (on) {
      for (int y = it.y0; y < yend; ++y) {
        const int64_t i = int64_t(y) * a.W + x;
        const int s = slot_of(it, a.labels[i]);
        if (s < 0) continue;
        const double rv = a.r[i];
#pragma unroll
        for (int j = 0; j < SLOTS; ++j)
          if (j == s) acc[j] += rv * rv;
      }
    }
    item_finish(a, it, acc, [&](int32_t c, double bb) {
      a.rho[c] = bb;
      const double bn = sqrt(bb);
      a.tol[c] = rtol * bn;
      a.iters[c] = 0;
      a.alpha[c] = 0.0;
      a.beta[c] = 0.0;
      a.brk[c] = 0;
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

// status "active" only while the initial norm pass counts arrivals; the
// finaliser of that pass sets the real state (ST_ACTIVE counts toward
// a.active only there).
__global__ void init_state_kernel(FillArgs a, const int32_t* __restrict__ comp_size, int C,
                                  int cg_max_iters) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    a.status[c] = comp_size[c] >= 2 ? ST_ACTIVE : ST_IDLE;
    a.iters[c] = 0;
    a.brk[c] = 0;
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
  float *x, *r, *p0, *p1, *q, *hw;
  uint8_t* imask;
  int32_t *slot_base, *nslots, *nitems_strip, *item_base, *strip_comps, *partial_comp,
      *partial_idx, *plist, *keys_sorted;
  Item* items;
  int32_t *comp_size, *comp_nparts, *comp_pstart, *comp_cnt, *iters, *cap, *active, *changed,
      *total, *total_items, *active_items, *nactive_items;
  double *partial, *rho, *alpha, *beta, *tol;
  uint8_t *status, *brk;
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
  w.r = c.take<float>(npix);
  w.p0 = c.take<float>(npix);
  w.p1 = c.take<float>(npix);
  w.q = c.take<float>(npix);
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
  w.partial = c.take<double>(P);
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
  w.brk = c.take<uint8_t>(C + 1);
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
                         w.x, w.r, w.p0, w.p1, w.q, w.comp_size)
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
  a.r = w.r;
  a.q = w.q;
  a.p0 = w.p0;
  a.p1 = w.p1;
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
  a.brk = w.brk;
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
    // occupancy variant (experiments): NI_FILL_MINB=3 gives 85 registers
    const char* mb = getenv("NI_FILL_MINB");
    const bool m3 = mb && atoi(mb) == 3;
    void* kfn = connectivity == 8 ? (m3 ? (void*)fill_cg_kernel<8, 3> : (void*)fill_cg_kernel<8, 4>)
                                  : (m3 ? (void*)fill_cg_kernel<4, 3> : (void*)fill_cg_kernel<4, 4>);
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

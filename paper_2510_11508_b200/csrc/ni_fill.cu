// Weighted fill passes -- the refill pass of solver.py:237-238 and the
// pixel-level baseline of pipeline.py:297-369 -- as ONE batched,
// unpreconditioned CG over every component of the partition, matrix-free on
// the pixel grid, run by ONE persistent kernel of independent worker warps.
// (The plain fill at z = 0 runs the multigrid-preconditioned solve of
// ni_mg.cu; this kernel also serves it behind NI_FILL_SOLVER=cg.)
//
// Per component c the reference solves (A^T W A) x = A^T W b with scipy's
// unpreconditioned CG (x0 = 0, stop when ||r|| < rtol ||b|| at the top of an
// iteration, cap max(cg_max_iters, n_c); solver.py:97-122).  Without edge
// weights (the fill at z = 0) every bilateral factor is 1/2
// (continuity.py:302-308): W_a = gamma_a^2 / 2 and A^T W A is the graph
// Laplacian of the intra-component valid edges with conductance c_ab = W_a +
// W_b; the EW variant takes per-edge weights (w_a, w_b) instead.  All
// components iterate together; each keeps its own alpha/beta/rho, stop test
// and cap, exactly like separate scipy solves.  The stencil is applied in
// difference form q_a = sum c_ab (p_a - p_b), so constants stay an exact
// null vector in float32.
//
// Data layout in HBM.  rows = B*H; pixel (y, x) lives at padded index
// (y + RM) * P + (x + XM) with zeroed margins, so no access needs a bounds
// check:
//   v[2]  : float4 {r, q, p, x} per pixel, double-buffered by iteration
//           parity (a sweep reads its neighbours' previous values while other
//           warps write the new ones)
//   hw    : float32 W_a = gamma_a^2 / 2 (EW: four forward conductances)
//   imask : uint8, bit k = forward edge k intra-component and valid,
//           bit 4+k = backward edge k (pixel - offset_k)
//   lab   : int32 labels (read by mixed items only)
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
// stops gets one last "flush" sweep that applies its pending x update; its
// final x then lives in the buffer of that sweep's parity.
//
// Work decomposition: strips of 30 x 30 centre pixels, never straddling two
// maps.  A warp processes a strip ("item") by streaming its 32 rows (lanes
// and rows 0 / 31 are the halo) through a per-warp shared-memory ring of row
// slots filled by cp.async several rows ahead, forming p' = r + beta p once
// per row and taking the horizontal neighbours by shuffles.  A CTA (one per
// SM) is 15 sweeping warps + 1 scheduler warp that claims items into
// per-worker mailboxes and retires finished ones; components sharing items
// iterate in lockstep "groups" whose batches are published through a ring
// (DESIGN.md s5b).  A strip touching several multi-pixel components becomes
// items of <= 2 components that read labels; a strip with one component is
// a "pure" item (singleton / invalid pixels carry r = q = p = x = 0).
//
// Reductions are deterministic: each item writes float64 partials per
// component (lane-local sums over rows, fixed xor tree over lanes); the last
// warp to arrive for a component (integer counter) sums the component's
// partials in plan order and updates its scalars.
// Algorithmic bytes per active pixel and iteration (pure items):
//   read r, q, p, x, hw (20 B) + imask (1 B); write r, q, p, x (16 B) => 37 B/px
// (halo rows/columns are re-read from L1/L2 and not counted).
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>

#include <cub/device/device_radix_sort.cuh>

#include "ni_common.cuh"

namespace cg = cooperative_groups;

namespace ni {

constexpr int SW = 30;     // strip width (lanes 1..30; lanes 0 / 31 are the halo)
#ifndef NI_SH
#define NI_SH 30
#endif
constexpr int SH = NI_SH;  // strip height (centre rows per item)
constexpr int SPX = SW * SH <= 1024 ? 1024 : 2048;  // padded pixels per strip (sort buffer)
constexpr int NT = 256;    // threads per CTA (8 warps)
constexpr int WPB = NT / 32;
constexpr int SLOTS = 2;  // components per item
constexpr int kPairMaps = 10;  // batches of at least this many maps pair components in items
constexpr int NDOT = 4;   // <p,q>, <r,q>, <q,q>, <r,r>
constexpr int XM = 16;    // left margin (columns)
constexpr int RM = 2;     // top margin (rows)
constexpr int RB = SH + 4;  // bottom margin (rows): every item streams SH + 2 rows

enum : uint8_t { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_CAPPED = 2, ST_IDLE = 3, ST_FLUSH = 4 };

// One work item: a strip and up to 2 of its components.
struct __align__(16) Item {
  int32_t x0, y0;  // top-left centre pixel of the strip (column of lane 1)
  int32_t pbase;   // first partial slot of this item
  int32_t flags;   // bits 0-7: components in the item (1..2); bit 8: pure strip
  int32_t comp[SLOTS];
  int32_t y1;  // end row of the strip (strips never straddle two maps)
  int32_t pad;
};

__device__ __forceinline__ int item_n(const Item& it) { return it.flags & 0xFF; }
__device__ __forceinline__ bool item_pure(const Item& it) { return (it.flags >> 8) & 1; }
__device__ __forceinline__ int item_n_flags(int32_t flags) { return flags & 0xFF; }

struct FillArgs {
  int rows, W, P;
  float4* v[2];
  const float* hw;        // fill: W_a = gamma_a^2 / 2 (c_ab = hw_a + hw_b)
  const float4* cf;       // EW passes: forward-edge conductances W_a + W_b, edges 0..3
  const uint8_t* imask;
  const int32_t* lab;  // padded labels
  // plan
  const Item* items;
  int nitems;
  const int32_t* comp_pstart;  // [C+1] partial range per component
  const int32_t* comp_plist;   // [P] partial indices grouped by component
  int32_t* comp_cnt;           // [C] arrival counters (zero between sweeps)
  double* partial;             // [P][NDOT]
  // dataflow schedule: components sharing an item form a "group" that
  // iterates in lockstep; groups advance independently (see fill_cg_kernel)
  int G;                       // groups
  const int32_t* cgrp;         // [C] group of a component
  const int32_t* gstart;       // [G+1] region of a group in active_items
  int32_t* active_items;       // [nitems] per-group lists of live items
  int32_t* gcnt;               // [G] live items of the group
  unsigned long long* gtk;     // [G] open batch: parity << 63 | n << 32 | next ticket
  int32_t* gdone;              // [G] items finished in the open batch
  int32_t* gchg;               // [G] a component of the group reached its final state
  unsigned long long* ring;    // [R] published batches: seq << 32 | group
  uint32_t R;                  // ring capacity (power of two)
  uint32_t* ring_tail;
  uint32_t* ring_hint;         // every ring entry below it is exhausted
  uint32_t* gseq;              // [G] ring position of the group's newest entry
  int32_t* gactive;            // groups with live items
  // admission window: at most `window` groups hold published batches at a
  // time (0: all), so their state can stay in L2; a retiring group admits
  // the next one (gnext) in group order
  int window;
  int32_t* gnext;
  int mb;  // mailbox slots the scheduler fills per worker (1..MB)
  // component state
  double* rho;     // exact <r_k, r_k> / then the rho_{k+1} estimate
  double* alpha;   // alpha of the last completed sweep
  double* beta;
  double* tol;
  int32_t* iters;
  int32_t* cap;
  uint8_t* status;
  uint8_t* final_status;  // status after the flush sweep
  uint8_t* xbuf;          // buffer holding the component's final x
};

// ----------------------------------------------------------------- setup

// Padded-layout setup: v[0] = {b, 0, 0, 0}, hw (fill) or the forward-edge
// conductances cf (EW: per-edge weights w_a / w_b given), imask, labels.
template <int CONN, int MODEL, bool EW>
__global__ void __launch_bounds__(256) prep_kernel(
    const int32_t* __restrict__ labels, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, const double* __restrict__ w_a,
    const double* __restrict__ w_b, int H, int W, int P, int64_t npix, float* __restrict__ hw,
    float4* __restrict__ cf, uint8_t* __restrict__ imask, int32_t* __restrict__ lab_p,
    float4* __restrict__ v0, int32_t* __restrict__ comp_size) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t lab = labels[i];
    const int u = int(i % W);
    const int64_t row = i / W;
    const int vloc = int(row % H);
    const int64_t o = (row + RM) * P + u + XM;  // padded index
    lab_p[o] = lab;
    if (lab < 0) continue;  // margins / invalid pixels stay zero
    {  // one atomic per distinct label of the warp (neighbours share labels)
      const unsigned peers = __match_any_sync(__activemask(), lab);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(comp_size + lab, __popc(peers));
    }
    // fill weights at z = 0: every bilateral factor is 1/2 (continuity.py:302-308)
    const double wself = 0.5 * (gamma[i] * gamma[i]);
    if (!EW) hw[o] = float(wself);
    float c[4] = {0.f, 0.f, 0.f, 0.f};
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
          const double wa = EW ? w_a[k * npix + i] : wself;
          const double wb = EW ? w_b[k * npix + i] : 0.5 * (gamma[j] * gamma[j]);
          const double oa = omega_a[k * npix + i];
          const double ob = MODEL == 0 ? -oa : omega_b[k * npix + i];
          b += wa * oa - wb * ob;  // A^T W b of rows 2e, 2e+1 (solver.py:83-93)
          c[k] = float(wa + wb);
        }
      }
      // backward edge (j -> i), j = i - offset_k: i is the "b" endpoint
      const int uj = u - du, vj = vloc - dv;
      if (uj >= 0 && uj < W && vj >= 0) {
        const int64_t j = i - int64_t(dv) * W - du;
        const uint8_t efj = eflags[j];
        if (((efj >> k) & (efj >> (4 + k)) & 1) && labels[j] == lab) {
          m |= uint8_t(1u << (4 + k));
          const double wj = EW ? w_a[k * npix + j] : 0.5 * (gamma[j] * gamma[j]);
          const double wi = EW ? w_b[k * npix + j] : wself;
          const double oa = omega_a[k * npix + j];
          const double ob = MODEL == 0 ? -oa : omega_b[k * npix + j];
          b += wi * ob - wj * oa;
        }
      }
    }
    imask[o] = m;
    if (EW) cf[o] = make_float4(c[0], c[1], c[2], c[3]);
    v0[o] = make_float4(float(b), 0.f, 0.f, 0.f);
  }
}

// Strip s of the grid: nsx strips across, nsym per map (the last one of a
// map may be short), map-major.
__device__ __forceinline__ void strip_rect(int s, int nsx, int nsym, int H, int& x0, int& y0,
                                           int& y1) {
  const int r = s / nsx, m = r / nsym;
  x0 = (s % nsx) * SW;
  y0 = m * H + (r % nsym) * SH;
  y1 = min(y0 + SH, (m + 1) * H);
}

// One CTA per strip: its distinct multi-pixel components, ascending.
__global__ void __launch_bounds__(NT) strip_comps_kernel(const int32_t* __restrict__ labels,
                                                         const int32_t* __restrict__ comp_size,
                                                         int H, int W, int nsx, int nsym,
                                                         int32_t* __restrict__ nslots,
                                                         int32_t* __restrict__ strip_comps) {
  __shared__ int32_t key[SPX];
  __shared__ int32_t wcount[WPB];
  const int strip = blockIdx.x, tid = threadIdx.x;
  int x0, y0, y1;
  strip_rect(strip, nsx, nsym, H, x0, y0, y1);
  for (int e = tid; e < SPX; e += NT) {
    int32_t lab = -1;
    if (e < SW * SH) {
      const int gx = x0 + (e % SW), gy = y0 + (e / SW);
      if (gx < W && gy < y1) {
        lab = labels[int64_t(gy) * W + gx];
        if (lab >= 0 && comp_size[lab] < 2) lab = -1;  // singletons never iterate (solver.py:220)
      }
    }
    key[e] = lab < 0 ? INT32_MAX : lab;
  }
  __syncthreads();
  // fast path: most strips hold a single component (or none) -- no sort
  {
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (int e = tid; e < SPX; e += NT) {
      const int32_t k = key[e];
      if (k != INT32_MAX) {
        lo = min(lo, k);
        hi = max(hi, k);
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    __shared__ int32_t wlo[WPB], whi[WPB];
    if ((tid & 31) == 0) {
      wlo[tid >> 5] = lo;
      whi[tid >> 5] = hi;
    }
    __syncthreads();
    lo = wlo[0];
    hi = whi[0];
#pragma unroll
    for (int w = 1; w < WPB; ++w) {
      lo = min(lo, wlo[w]);
      hi = max(hi, whi[w]);
    }
    if (lo == INT32_MAX || lo == hi) {  // block-uniform branch
      if (tid == 0) {
        if (lo != INT32_MAX) strip_comps[int64_t(strip) * SPX] = lo;
        nslots[strip] = lo == INT32_MAX ? 0 : 1;
      }
      return;
    }
  }
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
                                   const int32_t* __restrict__ strip_comps, int nstrips, int nsx, int nsym, int H,
                                   int per, Item* __restrict__ items, int32_t* __restrict__ partial_comp,
                                   int32_t* __restrict__ partial_idx,
                                   int32_t* __restrict__ comp_nparts) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nstrips; s += gridDim.x * blockDim.x) {
    const int ns = nslots[s];
    if (ns == 0) continue;
    const int pb = slot_base[s], ib = item_base[s];
    for (int k = 0; k * per < ns; ++k) {
      Item it;
      strip_rect(s, nsx, nsym, H, it.x0, it.y0, it.y1);
      it.pbase = pb + k * per;
      const int n = min(per, ns - k * per);
      it.flags = n | ((ns == 1 ? 1 : 0) << 8);
#pragma unroll
      for (int j = 0; j < SLOTS; ++j)
        it.comp[j] = j < n ? strip_comps[int64_t(s) * SPX + k * per + j] : -1;
      it.pad = 0;
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

__global__ void item_counts_kernel(const int32_t* __restrict__ nslots, int nstrips, int per,
                                   int32_t* __restrict__ nitems) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nstrips; s += gridDim.x * blockDim.x)
    nitems[s] = (nslots[s] + per - 1) / per;
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
template <int NSUM = SLOTS, class Fin>
__device__ __forceinline__ bool item_finish(const FillArgs& a, const Item& it,
                                            double (&acc)[SLOTS][NDOT], const bool* live, Fin fin) {
  const int lane = threadIdx.x & 31;
  const int n = item_n(it);
  double tot[SLOTS][NDOT];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int d = 0; d < NDOT; ++d) tot[s][d] = s < NSUM ? warp_sum(acc[s][d]) : 0.0;
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
  const bool ran = lastmask != 0;
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
  return ran;
}

// ---- the per-warp row stream (cp.async into a shared-memory ring)
//
// Every item is a stream of 32 rows (local rows 0..31 = real rows y0-1 ..
// y0+30) of its 32 columns (real x0-1 .. x0+30).  A warp's items follow each
// other in one continuous stream; local row j lives in ring slot j % NS
// (IROWS is a multiple of NS) and is copied LA rows ahead of its use, so the
// next item's first rows are in flight while the current item finishes.
// Copies are cp.async (LDGSTS): in-flight rows hold no registers.  Per row
// every lane copies 16 B of {r,q,p,x}; lanes 0-8 copy the hw window, lanes
// 9-17 the label window (mixed items only), lanes 18-20 the imask window.
#ifndef NI_NS
#define NI_NS 8
#endif
constexpr int NS = NI_NS;  // ring slots per warp
constexpr int IROWS = SH + 2;  // stream rows per item
constexpr int GR = 2;      // centre rows computed per step (between two waits)
constexpr int LA = NS - GR;  // rows in flight beyond the ones being derived
static_assert((NS & (NS - 1)) == 0 && IROWS % NS == 0, "ring slots must tile an item");
static_assert(SH % GR == 0 && (IROWS - 2 - LA) % GR == 0, "row steps must align");
static_assert(LA >= 2, "ring too small");

// Ring slot layouts (bytes).  Fill: {r,q,p,x}[32] | hw[36] | labels[36] |
// imask[48].  Edge-weighted passes (EW: refill, pixel baseline): {r,q,p,x}[32]
// | forward conductances float4[32] | labels[36] | imask[48].
template <bool EW>
struct Slot {
  static constexpr int V = 0, H = 512, C = 512;
  static constexpr int LAB = EW ? 1024 : 656;
  static constexpr int M = LAB + 144;
  static constexpr int BYTES = M + 48;
};

// A claimed item with its coefficients; the next item's lives in shared
// memory (one per warp) so it holds no registers while the current item runs.
struct Claim {
  Item item;
  float al[SLOTS], be[SLOTS];
  int32_t g, par, n, live;  // live: bit j = slot j is ACTIVE or FLUSH
  uint8_t st[SLOTS];
};
template <bool EW>
constexpr size_t ring_bytes() {
  return size_t(Slot<EW>::BYTES) * NS;
}
#ifndef NI_WORKERS
#define NI_WORKERS 15
#endif
constexpr int WORKERS = NI_WORKERS;          // sweeping warps per CTA (one CTA per SM)
constexpr int NT_FILL = (WORKERS + 1) * 32;  // + one scheduler warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, bool on) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
      " @p cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(dst),
      "l"(src), "r"(int(on))
      : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The copy side of a warp's row stream (per-lane source pointers).
struct Issuer {
  const char* v;    // this lane's 16 B of {r,q,p,x} in the next row
  const char* c;    // this lane's 16 B of forward conductances (EW passes)
  const char* aux;  // this lane's 16 B of hw / labels / imask in the next row
  uint32_t apitch;  // aux row pitch in bytes
  uint32_t adst;    // aux destination offset in a slot
  bool on, aon;     // off: past the last item / lane copies no aux bytes
};

template <bool EW>
__device__ __forceinline__ void issuer_start(const FillArgs& a, const Item& it, int par,
                                             Issuer& is) {
  using L = Slot<EW>;
  const int lane = threadIdx.x & 31;
  const int c0 = it.x0 - 1 + XM;  // padded column of lane 0
  const int64_t row0 = int64_t(it.y0 - 1 + RM) * a.P;
  const int ah = c0 & ~3, am = c0 & ~15;  // 16-B aligned windows
  is.v = reinterpret_cast<const char*>(a.v[par] + row0 + c0 + lane);
  is.on = true;
  if (EW) {
    is.c = reinterpret_cast<const char*>(a.cf + row0 + c0 + lane);
    if (lane < 9) {
      is.aux = reinterpret_cast<const char*>(a.lab + row0 + ah + 4 * lane);
      is.apitch = 4u * a.P;
      is.adst = L::LAB + 16 * lane;
      is.aon = !item_pure(it);
    } else {
      is.aux = reinterpret_cast<const char*>(a.imask + row0 + am + 16 * (lane - 9));
      is.apitch = a.P;
      is.adst = L::M + 16 * (lane - 9);
      is.aon = lane < 12;
    }
    return;
  }
  if (lane < 9) {
    is.aux = reinterpret_cast<const char*>(a.hw + row0 + ah + 4 * lane);
    is.apitch = 4u * a.P;
    is.adst = L::H + 16 * lane;
    is.aon = true;
  } else if (lane < 18) {
    is.aux = reinterpret_cast<const char*>(a.lab + row0 + ah + 4 * (lane - 9));
    is.apitch = 4u * a.P;
    is.adst = L::LAB + 16 * (lane - 9);
    is.aon = !item_pure(it);
  } else {
    is.aux = reinterpret_cast<const char*>(a.imask + row0 + am + 16 * (lane - 18));
    is.apitch = a.P;
    is.adst = L::M + 16 * (lane - 18);
    is.aon = lane < 21;
  }
}

// Copy the issuer's next row into ring slot `j % NS` (one commit group per
// row in every lane, empty once the stream is off).
template <bool EW>
__device__ __forceinline__ void issue_row(uint32_t ring, int j, Issuer& is, uint32_t vpitch) {
  using L = Slot<EW>;
  const int lane = threadIdx.x & 31;
  const uint32_t slot = ring + uint32_t(j & (NS - 1)) * L::BYTES;
  cp_async16_if(slot + L::V + 16 * lane, is.v, is.on);
  if (EW) {
    cp_async16_if(slot + L::C + 16 * lane, is.c, is.on);
    is.c += vpitch;
  }
  cp_async16_if(slot + is.adst, is.aux, is.on && is.aon);
  cp_commit();
  is.v += vpitch;
  is.aux += is.apitch;
}

// A row of the compute ring: r_k, p_k = r_k + beta p_{k-1}, x_k formed with
// the pixel's own component (only intra-component neighbours are ever read,
// and those share the centre's alpha and beta), plus the left / right
// neighbours' p' and hw (warp shuffles; lanes 0 / 31 are the halo).
// EW rows carry the pixel's forward conductances c0..c3 and the backward
// ones it needs from its neighbours: c0l (left pixel's c0), c1r (right
// pixel's c1), c3l (left pixel's c3).
template <bool EW>
struct RowT {
  float pn, h, pl, pr, hl, hr, rn, xn;
  uint32_t m;  // imask | (slot + 1) << 8
};
template <>
struct RowT<true> {
  float pn, pl, pr, rn, xn;
  float c0, c1, c2, c3, c0l, c1r, c3l;
  uint32_t m;  // imask | (slot + 1) << 8
};

struct Cur {  // the current item, in registers
  int32_t x0, y0, y1, flags, pbase, g, par, n, live;
  int32_t comp[SLOTS];
  float al[SLOTS], be[SLOTS];
};

__device__ __forceinline__ void load_cur(const Claim& c, Cur& k) {
  k.x0 = c.item.x0;
  k.y0 = c.item.y0;
  k.y1 = c.item.y1;
  k.flags = c.item.flags;
  k.pbase = c.item.pbase;
  k.g = c.g;
  k.par = c.par;
  k.n = c.n;
  k.live = c.live;
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) {
    k.comp[j] = c.item.comp[j];
    k.al[j] = c.al[j];
    k.be[j] = c.be[j];
  }
}

// Shared-memory loads by 32-bit shared address (register + immediate
// addressing; a generic pointer into the ring re-derives the shared window
// every row).  volatile keeps them after the cp.async wait that precedes them.
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// This lane's shared addresses in ring slot 0 (a slot is + slot * BYTES).
struct LaneOfs {
  uint32_t v;  // {r,q,p,x}
  uint32_t c;  // forward conductances (EW)
  uint32_t h;  // hw
  uint32_t l;  // label
  uint32_t m;  // imask byte
};

template <bool PURE, bool EW>
__device__ __forceinline__ RowT<EW> derive(uint32_t slot, const LaneOfs& o_, const Cur& k) {
  const float4 v = lds_f4(slot + o_.v);
  float al = k.al[0], be = k.be[0];
  int s = 0;
  if (!PURE) {
    const int32_t lab = lds_s32(slot + o_.l);
    s = lab == k.comp[0] ? 0 : (item_n_flags(k.flags) > 1 && lab == k.comp[1] ? 1 : -1);
    al = s == 0 ? k.al[0] : (s == 1 ? k.al[1] : 0.f);
    be = s == 0 ? k.be[0] : (s == 1 ? k.be[1] : 0.f);
  }
  RowT<EW> o;
  o.rn = fmaf(-al, v.y, v.x);
  o.pn = fmaf(be, v.z, o.rn);
  o.xn = fmaf(al, v.z, v.w);
  o.m = lds_u8(slot + o_.m) | (uint32_t(s + 1) << 8);
  o.pl = __shfl_up_sync(0xffffffffu, o.pn, 1);
  o.pr = __shfl_down_sync(0xffffffffu, o.pn, 1);
  if constexpr (EW) {
    const float4 c = lds_f4(slot + o_.c);
    o.c0 = c.x;
    o.c1 = c.y;
    o.c2 = c.z;
    o.c3 = c.w;
    o.c0l = __shfl_up_sync(0xffffffffu, c.x, 1);
    o.c1r = __shfl_down_sync(0xffffffffu, c.y, 1);
    o.c3l = __shfl_up_sync(0xffffffffu, c.w, 1);
  } else {
    o.h = lds_f32(slot + o_.h);
    o.hl = __shfl_up_sync(0xffffffffu, o.h, 1);
    o.hr = __shfl_down_sync(0xffffffffu, o.h, 1);
  }
  return o;
}

#ifndef NI_FILL_STATS
#define NI_FILL_STATS 0
#endif
#if NI_FILL_STATS
// debug counters (variant build): 0 worker cycles, 1 worker idle (empty
// mailbox), 2 worker waits for a finish slot, 3 items, 4 scheduler cycles,
// 5 scheduler retire cycles, 6 scheduler claim cycles, 7 claims
__device__ unsigned long long g_fill_stats[8];
#define NI_STAT(i, v) atomicAdd(&g_fill_stats[i], (unsigned long long)(v))
#else
#define NI_STAT(i, v) ((void)0)
#endif

#ifndef NI_IDLE_NS
#define NI_IDLE_NS 64  // a worker's poll interval on an empty mailbox
#endif

// ---- warp roles
//
// A CTA is WORKERS sweeping warps plus one scheduler warp.  The scheduler
// claims items for the workers (into a per-worker mailbox in shared memory)
// and retires finished items (partials, per-component finalisers, batch
// accounting), so a worker only ever streams rows: the dependent global
// round trips of claiming and retiring overlap the sweeps instead of
// stalling them.
#ifndef NI_MB
#define NI_MB 2
#endif
#ifndef NI_FQ
#define NI_FQ 4
#endif
constexpr int MB = NI_MB;  // claimed items per worker mailbox
constexpr int FQ = NI_FQ;  // finished-item records per worker
static_assert(32 / NI_WORKERS >= 1, "one record per lane and wave");
static_assert(NI_MB * NI_WORKERS <= 32, "one claim target per lane");

struct Mailbox {  // scheduler -> worker (single producer, single consumer)
  Claim slot[MB];
  int head;  // items the worker has started (worker-owned)
  int tail;  // items the scheduler has posted (scheduler-owned)
  int pad[2];
};

struct FinishRec {
  double sum[SLOTS][NDOT];  // warp-summed <p,q>, <r,q>, <q,q>, <r,r> per slot
  int32_t comp[SLOTS];
  int32_t pbase, nslot, g, n, par, live;
};

struct FinishBox {  // worker -> scheduler (single producer, single consumer)
  FinishRec rec[FQ];
  int head;  // records retired (scheduler-owned)
  int tail;  // records posted (worker-owned)
  int pad[2];
};

struct CtaShared {
  Mailbox mb[WORKERS];
  FinishBox fb[WORKERS];
  int done;  // set by the scheduler once every group retired
  int pad[3];
};

template <bool EW>
constexpr size_t smem_bytes() {
  return ring_bytes<EW>() * WORKERS + sizeof(CtaShared);
}

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
// A poll whose outcome steers the whole warp: lane 0's read, broadcast, so
// the lanes can never disagree (a mailbox tail posted between two lanes'
// reads would otherwise split the warp in front of full-mask shuffles).
__device__ __forceinline__ int vload_warp(const int* p) {
  return __shfl_sync(0xffffffffu, vload(p), 0);
}
__device__ __forceinline__ void vstore(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

// ---- the batch scheduler
//
// A group's open batch is one 64-bit word: parity << 63 | n << 32 | ticket.
// Claiming is one atomicAdd on it: tickets t < n of the returned word are
// items of that batch, whatever ring entry led there.  Published batches
// are announced in a ring (seq << 32 | group); the scheduler probes 32
// entries from the hint at once and takes the first open one, so batches
// drain in publication order and the hint only passes exhausted entries.
// Ring entries are read relaxed: the group word (gtk) and newest-entry
// position (gseq) are then read through L2 (ld.cg) at addresses computed from
// the entry, so they are fetched after it and see what publish() wrote before
// its release store.  (An acquire load here costs an L1 invalidation per
// probe: 3-6 % of the fill.)
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Claim up to `want` (<= 32) items of one open batch with a single ticket
// atomic; lane j < got writes item t + j into *dst[j] (shared memory).
// Returns how many (0: no batch is open).
__device__ __noinline__ int claim_items(const FillArgs& a, int want, Claim* const* dst) {
  const int lane = threadIdx.x & 31;
  uint32_t h = *reinterpret_cast<const volatile uint32_t*>(a.ring_hint);
  for (int round = 0; round < 64; ++round) {
    const uint32_t p = h + lane;
    const unsigned long long e = ld_relaxed_u64(a.ring + (p & (a.R - 1)));
    const uint32_t seq = uint32_t(e >> 32);
    const bool pub = seq == p;
    const bool stale = int32_t(seq - p) > 0;  // lapped: long exhausted
    const int32_t g = int32_t(e & 0xffffffffu);
    bool open = false;
    int key = -1;  // priority: the batch's item count (larger groups first)
    // An entry that is not its group's newest one is exhausted: its batch
    // completed before the group published again.  (Reading the group's
    // current batch through it instead made old entries stand in for newer
    // batches; with the largest-first priority such stand-ins could keep a
    // slightly smaller group's batch unclaimed until the ring lapped it.)
    {
      const int32_t gi = pub ? g : 0;  // both loads in flight at once
      const uint32_t last = __ldcg(a.gseq + gi);
      const unsigned long long w = __ldcg(a.gtk + gi);
      if (pub && last == p) {
        const int n = int((w >> 32) & 0x7fffffffu);
        open = int(w & 0xffffffffu) < n;
        if (open) key = n;
      }
    }
    const unsigned openm = __ballot_sync(0xffffffffu, open);
    const unsigned donem = __ballot_sync(0xffffffffu, (pub && !open) || stale);
    const int lead = __ffs(~donem) - 1;  // leading exhausted entries (-1: all 32)
    const int k = lead < 0 ? 32 : lead;
    if (lane == 0 && k > 0) atomicCAS(a.ring_hint, h, h + k);
    if (openm) {
      // the open batch of the largest group in the window: the largest
      // components take the most iterations, so serving them first keeps
      // the critical path short when few groups remain
      int best = key, l = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ol = __shfl_xor_sync(0xffffffffu, l, o);
        if (ob > best || (ob == best && ol < l)) {
          best = ob;
          l = ol;
        }
      }
      const int32_t gg = __shfl_sync(0xffffffffu, g, l);
      unsigned long long w = 0;
      int32_t gs = 0;
      if (lane == 0) w = atomicAdd(a.gtk + gg, static_cast<unsigned long long>(want));
      if (lane == 1) gs = __ldcg(a.gstart + gg);
      w = __shfl_sync(0xffffffffu, w, 0);
      gs = __shfl_sync(0xffffffffu, gs, 1);
      const int32_t t = int32_t(w & 0xffffffffu), n = int32_t((w >> 32) & 0x7fffffffu);
      const int got = max(0, min(want, n - t));
      if (got > 0) {
        // the batch's coefficients were published before its word
        if (lane < got) {
          const int32_t k = __ldcg(a.active_items + gs + t + lane);
          const Item it = a.items[k];
          const int ni = item_n(it);
          int live = 0;
          Claim& cj = *dst[lane];
#pragma unroll
          for (int j = 0; j < SLOTS; ++j) {
            float al = 0.f, be = 0.f;
            uint8_t st = ST_IDLE;
            if (j < ni) {
              const int32_t cc = it.comp[j];
              st = __ldcg(a.status + cc);
              al = float(__ldcg(a.alpha + cc));
              be = float(__ldcg(a.beta + cc));
              if (st == ST_ACTIVE || st == ST_FLUSH) live |= 1 << j;
            }
            cj.al[j] = al;
            cj.be[j] = be;
            cj.st[j] = st;
          }
          cj.item = it;
          cj.g = gg;
          cj.par = int32_t(w >> 63);
          cj.n = n;
          cj.live = live;
        }
        __syncwarp();
        return got;
      }
      continue;  // lost the race for the last tickets: probe again
    }
    if (donem != 0xffffffffu) return 0;  // reached the unpublished tail
    h += 32;
  }
  return 0;
}

// Announce group g's next batch (lane 0).
#if NI_FILL_STATS
constexpr int kTraceG = 256, kTraceI = 4096;
__device__ unsigned long long g_pub_trace[kTraceG * kTraceI];
__device__ int g_pub_n[kTraceG];
#endif

__device__ __forceinline__ void publish(const FillArgs& a, int32_t g, int par, int32_t n) {
#if NI_FILL_STATS
  if (g < kTraceG) {
    const int idx = atomicAdd(&g_pub_n[g], 1);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (idx < kTraceI) g_pub_trace[g * kTraceI + idx] = t | (static_cast<unsigned long long>(n) << 48);
  }
#endif
  a.gdone[g] = 0;
  __threadfence();
  atomicExch(a.gtk + g, (static_cast<unsigned long long>(par) << 63) |
                            (static_cast<unsigned long long>(n) << 32));
  __threadfence();
  const uint32_t p = atomicAdd(a.ring_tail, 1u);
  a.gseq[g] = p;  // ordered before the entry by its release store
  const unsigned long long e = (static_cast<unsigned long long>(p) << 32) | uint32_t(g);
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.ring + (p & (a.R - 1))), "l"(e)
               : "memory");
}

__device__ __forceinline__ bool item_live(const FillArgs& a, int32_t k) {
  const Item it = a.items[k];
  const int n = item_n(it);
  bool act = false;
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
    if (j < n) {
      const uint8_t st = __ldcg(a.status + it.comp[j]);
      if (st == ST_ACTIVE || st == ST_FLUSH) act = true;
    }
  return act;
}

// A group retired under an admission window: publish the first batch of the
// next group that has live items (lane 0).
__device__ void admit_next(const FillArgs& a) {
  for (;;) {
    const int32_t g = atomicAdd(a.gnext, 1);
    if (g >= a.G) return;
    const int32_t n = __ldcg(a.gcnt + g);
    if (n > 0) {
      publish(a, g, 0, n);
      return;
    }
  }
}

// The warp that retires a group's batch: drop items whose components are
// all final (in-place stable compaction), then publish the next batch or
// retire the group.
__device__ __noinline__ void advance_group(const FillArgs& a, int32_t g, int par) {
  const int lane = threadIdx.x & 31;
  __threadfence();
  int32_t n = __ldcg(a.gcnt + g);
  if (__ldcg(a.gchg + g)) {
    int32_t* list = a.active_items + __ldcg(a.gstart + g);
    int32_t out = 0;
    constexpr int U = 8;  // independent loads in flight per lane
    for (int b = 0; b < n; b += 32 * U) {
      int32_t kk[U];
      bool keep[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = b + 32 * u + lane;
        kk[u] = i < n ? __ldcg(list + i) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) keep[u] = kk[u] >= 0 && item_live(a, kk[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned m = __ballot_sync(0xffffffffu, keep[u]);
        if (keep[u]) list[out + __popc(m & ((1u << lane) - 1))] = kk[u];
        out += __popc(m);
      }
    }
    n = out;
    if (lane == 0) {
      a.gcnt[g] = n;
      a.gchg[g] = 0;
    }
  }
  if (lane == 0) {
    if (n > 0) {
      publish(a, g, par ^ 1, n);
    } else {
      atomicSub(a.gactive, 1);
      if (a.window > 0) admit_next(a);
    }
  }
  __syncwarp();
}

// Per-component scalar update once all of its items reported (one lane).
__device__ __forceinline__ void finalize_component(const FillArgs& a, int32_t c, const double* d,
                                                   int par) {
  if (__ldcg(a.status + c) == ST_FLUSH) {  // the pending update is applied
    a.status[c] = __ldcg(a.final_status + c);
    a.xbuf[c] = uint8_t(par ^ 1);
    a.gchg[a.cgrp[c]] = 1;
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
  } else {
    a.beta[c] = rho1 / rr;
    a.rho[c] = rho1;
  }
}

// Retire up to 32 finished items at once, one per lane (lane < cnt holds
// `r`): partials, arrival counts, the finalisers of components whose last
// item this was (in plan order, warp-cooperative), then batch accounting.
__device__ void retire_items(const FillArgs& a, const FinishRec& r, int cnt) {
  const int lane = threadIdx.x & 31;
  const bool mine = lane < cnt;
  // (1) partials of live slots
  if (mine) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
      if (s < r.nslot && ((r.live >> s) & 1)) {
        double* dst = a.partial + size_t(r.pbase + s) * NDOT;
#pragma unroll
        for (int d = 0; d < NDOT; ++d) dst[d] = r.sum[s][d];
      }
  }
  __threadfence();
  // (2) arrivals; a lane whose item completes a component reports it
  unsigned lastbits = 0;
  if (mine) {
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
      if (s < r.nslot && ((r.live >> s) & 1)) {
        const int32_t c = r.comp[s];
        const int32_t np = __ldcg(a.comp_pstart + c + 1) - __ldcg(a.comp_pstart + c);
        if (atomicAdd(a.comp_cnt + c, 1) == np - 1) lastbits |= 1u << s;
      }
  }
  // (3) finalisers, one component at a time over the whole warp
  unsigned todo = __ballot_sync(0xffffffffu, lastbits != 0);
  const bool any_fin = todo != 0;
  if (any_fin) __threadfence();
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const unsigned bits = __shfl_sync(0xffffffffu, lastbits, src);
    const int par = __shfl_sync(0xffffffffu, r.par, src);
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (!((bits >> s) & 1)) continue;
      const int32_t c = __shfl_sync(0xffffffffu, r.comp[s], src);
      const int32_t q0 = __ldcg(a.comp_pstart + c), q1 = __ldcg(a.comp_pstart + c + 1);
      double sum[NDOT] = {0.0, 0.0, 0.0, 0.0};
      for (int j = q0 + lane; j < q1; j += 32) {
        const double* p = a.partial + size_t(__ldcg(a.comp_plist + j)) * NDOT;
#pragma unroll
        for (int d = 0; d < NDOT; ++d) sum[d] += __ldcg(p + d);
      }
#pragma unroll
      for (int d = 0; d < NDOT; ++d) sum[d] = warp_sum(sum[d]);
      if (lane == 0) {
        finalize_component(a, c, sum, par);
        a.comp_cnt[c] = 0;
      }
      __syncwarp();
    }
  }
  if (any_fin) __threadfence();
  // (4) batch accounting; the item that completes a batch advances its group
  bool glast = false;
  if (mine) glast = atomicAdd(a.gdone + r.g, 1) == r.n - 1;
  unsigned adv = __ballot_sync(0xffffffffu, glast);
  while (adv) {
    const int src = __ffs(adv) - 1;
    adv &= adv - 1;
    advance_group(a, __shfl_sync(0xffffffffu, r.g, src), __shfl_sync(0xffffffffu, r.par, src));
  }
}

// The scheduler warp of a CTA.
__device__ void scheduler_loop(const FillArgs& a, CtaShared& sh) {
  const int lane = threadIdx.x & 31;
  __shared__ Claim* targets[32];
#if NI_FILL_STATS
  const long long t_start = clock64();
  long long t_ret = 0, t_claim = 0, n_claims = 0;
#endif
  for (;;) {
    bool busy = false;
#if NI_FILL_STATS
    const long long t0 = clock64();
#endif
    // -- retire finished items (lane l < WORKERS looks at worker l's box)
    int pend = 0, fh = 0;
    if (lane < WORKERS) {
      fh = vload(&sh.fb[lane].head);
      // at most 32 records per wave (one per lane)
      pend = min(vload(&sh.fb[lane].tail) - fh, 32 / WORKERS);
    }
    // one record per lane: exclusive prefix over the workers' pending counts
    int incl = pend;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total > 0) {
      busy = true;
      __threadfence_block();
      // lane j takes record j: find its worker by the prefix sums
      int w = 0, base = 0;
#pragma unroll
      for (int l = 0; l < WORKERS; ++l) {
        const int in = __shfl_sync(0xffffffffu, incl, l);
        const int ex = in - __shfl_sync(0xffffffffu, pend, l);
        if (lane >= ex && lane < in) {
          w = l;
          base = ex;
        }
      }
      FinishRec r;
      if (lane < total) {
        const int h0 = vload(&sh.fb[w].head);
        r = sh.fb[w].rec[(h0 + lane - base) % FQ];
      }
      retire_items(a, r, total);
      __syncwarp();
      if (lane < WORKERS && pend > 0) vstore(&sh.fb[lane].head, fh + pend);
    }
#if NI_FILL_STATS
    const long long t1 = clock64();
    t_ret += t1 - t0;
#endif
    // -- keep every mailbox full
    int need = 0, mt = 0;
    if (lane < WORKERS) {
      mt = vload(&sh.mb[lane].tail);
      need = max(0, a.mb - (mt - vload(&sh.mb[lane].head)));
    }
    // claim targets, slot-major: the first free slot of every worker, then
    // the second ones, so a short claim feeds the emptiest mailboxes first
    static_assert(MB <= 2, "target order below is written for at most two mailbox slots");
    const unsigned m0 = __ballot_sync(0xffffffffu, need > 0);
    const unsigned m1 = __ballot_sync(0xffffffffu, need > 1);
    const unsigned below = (1u << lane) - 1;
    const int pos0 = __popc(m0 & below), pos1 = __popc(m0) + __popc(m1 & below);
    const int want = __popc(m0) + __popc(m1);
    if (want > 0) {
      if (need > 0) targets[pos0] = &sh.mb[lane].slot[mt % MB];
      if (need > 1) targets[pos1] = &sh.mb[lane].slot[(mt + 1) % MB];
      __syncwarp();
      const int got = claim_items(a, want, targets);
#if NI_FILL_STATS
      t_claim += clock64() - t1;
      n_claims += got > 0;
#endif
      if (got > 0) {
        busy = true;
        __threadfence_block();
        if (lane < WORKERS) {
          const int mine = (need > 0 && pos0 < got) + (need > 1 && pos1 < got);
          if (mine > 0) vstore(&sh.mb[lane].tail, mt + mine);
        }
      }
    }
    if (!busy) {
      if (vload_warp(reinterpret_cast<const int*>(a.gactive)) == 0) {
        // every group retired: nothing will be claimed or posted any more
        if (lane == 0) vstore(&sh.done, 1);
#if NI_FILL_STATS
        if (lane == 0) {
          NI_STAT(4, clock64() - t_start);
          NI_STAT(5, t_ret);
          NI_STAT(6, t_claim);
          NI_STAT(7, n_claims);
        }
#endif
        return;
      }
      __nanosleep(128);
    }
    __syncwarp();
  }
}

// Per-item state of a worker's sweep.
struct Sweep {
  uint32_t vdst;   // this lane's {r,q,p,x} destination in ring slot 0
  uint32_t cdst;   // this lane's conductance destination in ring slot 0 (EW)
  uint32_t adst;   // this lane's aux destination in ring slot 0
  float4* orow;    // this lane's output pixel in the next centre row
  LaneOfs lo;      // this lane's shared read addresses in ring slot 0
  int nrows;
  bool center;
};

// Copy the issuer's next row into the ring slot at byte offset `off`.
template <bool EW>
__device__ __forceinline__ void issue_row_c(const Sweep& w, uint32_t off, Issuer& is,
                                            uint32_t vpitch) {
  cp_async16_if(w.vdst + off, is.v, is.on);
  if (EW) {
    cp_async16_if(w.cdst + off, is.c, is.on);
    is.c += vpitch;
  }
  cp_async16_if(w.adst + off, is.aux, is.on && is.aon);
  cp_commit();
  is.v += vpitch;
  is.aux += is.apitch;
}

// One step of a sweep: centre rows g+1, g+2 (GR = 2), with GB = g % 4 known
// at compile time so that the compute-ring indices are constants (row r
// lives in der[r % 4]).  The ring-slot byte offsets of the two rows issued
// (g+2+LA, g+3+LA) and the two rows derived (g+2, g+3) come from the caller
// as register + immediate values (see sweep_item).
template <int CONN, bool PURE, bool EW, int GB>
__device__ __forceinline__ void sweep_step(const FillArgs& a, Sweep& w, Issuer& is,
                                           uint32_t vpitch, RowT<EW> (&der)[4],
                                           double (&acc)[SLOTS][NDOT], int g, uint32_t oi0,
                                           uint32_t oi1, uint32_t od0, uint32_t od1,
                                           const Cur& k) {
  static_assert(GR == 2, "the step body is written for two rows");
  issue_row_c<EW>(w, oi0, is, vpitch);
  issue_row_c<EW>(w, oi1, is, vpitch);
  cp_wait<LA>();  // rows up to g+3 have landed
  __syncwarp();
  der[(GB + 2) & 3] = derive<PURE, EW>(od0, w.lo, k);
  der[(GB + 3) & 3] = derive<PURE, EW>(od1, w.lo, k);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int L = g + u + 1;  // centre local row
    const RowT<EW>& U = der[(GB + u) & 3];
    const RowT<EW>& C = der[(GB + u + 1) & 3];
    const RowT<EW>& D = der[(GB + u + 2) & 3];
    const float pa = C.pn;
    const uint32_t m = C.m;
    float q = 0.f;
    if constexpr (EW) {
      // per-edge conductances: forward ones are the pixel's own, backward
      // ones the forward conductance of the neighbour the edge starts at
#define NI_C(bit, pp, cc) q = ((m >> (bit)) & 1u) ? fmaf(cc, pa - (pp), q) : q
      if (CONN == 8) {
        NI_C(0, C.pr, C.c0);   // (+1, 0)
        NI_C(1, D.pl, C.c1);   // (-1,+1)
        NI_C(2, D.pn, C.c2);   // ( 0,+1)
        NI_C(3, D.pr, C.c3);   // (+1,+1)
        NI_C(4, C.pl, C.c0l);  // (-1, 0): left pixel's (+1, 0)
        NI_C(5, U.pr, U.c1r);  // (+1,-1): up-right pixel's (-1,+1)
        NI_C(6, U.pn, U.c2);   // ( 0,-1): up pixel's (0,+1)
        NI_C(7, U.pl, U.c3l);  // (-1,-1): up-left pixel's (+1,+1)
      } else {
        NI_C(0, C.pr, C.c0);   // (+1, 0)
        NI_C(1, D.pn, C.c1);   // ( 0,+1)
        NI_C(4, C.pl, C.c0l);  // (-1, 0)
        NI_C(5, U.pn, U.c1);   // ( 0,-1)
      }
#undef NI_C
    } else {
    const float ha = C.h;
#define NI_E(bit, pp, hh) q = ((m >> (bit)) & 1u) ? fmaf(ha + (hh), pa - (pp), q) : q
    if (CONN == 8) {
      NI_E(0, C.pr, C.hr);  // (+1, 0)
      NI_E(1, D.pl, D.hl);  // (-1,+1)
      NI_E(2, D.pn, D.h);   // ( 0,+1)
      NI_E(3, D.pr, D.hr);  // (+1,+1)
      NI_E(4, C.pl, C.hl);  // (-1, 0)
      NI_E(5, U.pr, U.hr);  // (+1,-1)
      NI_E(6, U.pn, U.h);   // ( 0,-1)
      NI_E(7, U.pl, U.hl);  // (-1,-1)
    } else {
      NI_E(0, C.pr, C.hr);  // (+1, 0)
      NI_E(1, D.pn, D.h);   // ( 0,+1)
      NI_E(4, C.pl, C.hl);  // (-1, 0)
      NI_E(5, U.pn, U.h);   // ( 0,-1)
    }
#undef NI_E
    }
    // pure: every centre pixel is the component's or zero (invalid /
    // singleton pixels carry r = q = p = x = 0 and stay 0); mixed: only
    // pixels of a live slot are written.  Dots are summed for every slot and
    // ignored for a flushing one.
    const int s = PURE ? 0 : int(m >> 8) - 1;  // -1: pixel not in this item
    bool mine = w.center && L <= w.nrows;
    if (!PURE) mine = mine && s >= 0 && ((k.live >> s) & 1);
    if (mine) __stcg(w.orow, make_float4(C.rn, q, pa, C.xn));
    // branch-free dots: a pixel outside the item contributes fma(0, 0, acc)
#pragma unroll
    for (int j = 0; j < (PURE ? 1 : SLOTS); ++j) {
      const bool on = mine && (PURE || j == s);
      const double dp = on ? pa : 0.f, dq = on ? q : 0.f, dr = on ? C.rn : 0.f;
      acc[j][0] = fma(dp, dq, acc[j][0]);
      acc[j][1] = fma(dr, dq, acc[j][1]);
      acc[j][2] = fma(dq, dq, acc[j][2]);
      acc[j][3] = fma(dr, dr, acc[j][3]);
    }
    w.orow += a.P;
  }
}

// One CG sweep over one item (see the header), by a worker warp.  On entry
// the stream holds this item's rows 0..LA-1 (issued); as its last rows are
// issued the worker peeks its mailbox for the next item (nx) and starts that
// item's rows.  The warp-summed dots go to the scheduler as a FinishRec.
template <int CONN, bool PURE, bool EW>
__device__ __forceinline__ void sweep_item(const FillArgs& a, const unsigned char* ring,
                                           Mailbox& mb, int mbh, const Claim*& nx, Issuer& is,
                                           const Cur& k, bool& has_next, FinishBox& fb,
                                           int& fbt) {
  constexpr int GSW = IROWS - 2 - LA;  // first step that issues the next item's rows
  static_assert(SH % 4 == 2 && GSW % 4 == 0 && GSW < SH - 2 && GSW >= 0,
                "the unrolled step schedule below assumes these shapes");
  const int lane = threadIdx.x & 31;
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t vpitch = 16u * a.P;
  Sweep w;
  const int xr = k.x0 - 1 + lane;  // real column of this lane
  w.center = lane >= 1 && lane <= SW && xr < a.W;
  const int c0 = k.x0 - 1 + XM;
  {
    using L = Slot<EW>;
    const int dh = c0 & 3, dm = c0 & 15;  // offsets of the hw / label and imask windows
    w.lo.v = L::V + 16 * lane;
    w.lo.c = L::C + 16 * lane;
    w.lo.h = L::H + 4 * (dh + lane);
    w.lo.l = L::LAB + 4 * (dh + lane);
    w.lo.m = L::M + dm + lane;
  }
  w.orow = a.v[k.par ^ 1] + int64_t(k.y0 + RM) * a.P + (xr + XM);  // centre row 1
  w.nrows = k.y1 - k.y0;  // centre rows (local rows 1..nrows)
  w.vdst = ring_s + Slot<EW>::V + 16 * lane;
  w.cdst = ring_s + Slot<EW>::C + 16 * lane;
  w.adst = ring_s + is.adst;
  double acc[SLOTS][NDOT];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
#pragma unroll
    for (int d = 0; d < NDOT; ++d) acc[j][d] = 0.0;
  has_next = false;
  // Ring slot of local row j: j % NS.  With LA = NS - 2 a step at row g
  // (g % 4 == 0) issues rows g+NS, g+NS+1 into the slots of rows g, g+1 and
  // derives rows g+2, g+3; the next step (g+2) issues into the slots of g+2,
  // g+3 and derives g+4, g+5, which sit in the next 4-slot block of the ring.
  // hb = the byte offset of the block holding row g and hb2 that of the next
  // one, so every slot is hb or hb2 plus a compile-time multiple of BYTES.
  static_assert(LA == NS - 2 && NS % 4 == 0, "slot schedule below assumes LA = NS - 2");
  constexpr uint32_t B = Slot<EW>::BYTES;
  // rows LA and LA+1; rows 0 and 1 have landed once at most LA younger
  // row groups are pending
  issue_row_c<EW>(w, LA * B, is, vpitch);
  issue_row_c<EW>(w, (LA + 1) * B, is, vpitch);
  cp_wait<LA>();
  __syncwarp();
  RowT<EW> der[4];  // row r of the item lives in der[r % 4]
  der[0] = derive<PURE, EW>(ring_s, w.lo, k);
  der[1] = derive<PURE, EW>(ring_s + B, w.lo, k);
#pragma unroll 1
  for (int g = 0; g < SH - 2; g += 4) {
    if (g == GSW) {  // the stream moves on to the next item with the rows issued from here on
      has_next = mbh < vload_warp(&mb.tail);
      if (has_next) {
        __threadfence_block();
        nx = &mb.slot[mbh % MB];
        issuer_start<EW>(a, nx->item, nx->par, is);
      } else {
        is.on = false;
      }
    }
    const uint32_t hb = uint32_t(g & (NS - 4)) * B;
    const uint32_t hb2 = hb + 4 * B == NS * B ? 0u : hb + 4 * B;
    sweep_step<CONN, PURE, EW, 0>(a, w, is, vpitch, der, acc, g, hb, hb + B,
                                  ring_s + hb + 2 * B, ring_s + hb + 3 * B, k);
    sweep_step<CONN, PURE, EW, 2>(a, w, is, vpitch, der, acc, g + 2, hb + 2 * B, hb + 3 * B,
                                  ring_s + hb2, ring_s + hb2 + B, k);
  }
  {
    constexpr uint32_t hb = uint32_t((SH - 2) & (NS - 4)) * B;
    sweep_step<CONN, PURE, EW, 0>(a, w, is, vpitch, der, acc, SH - 2, hb, hb + B,
                                  ring_s + hb + 2 * B, ring_s + hb + 3 * B, k);
  }
  // post the item's dots (fixed xor tree over lanes) for the scheduler
  constexpr int NS_ = PURE ? 1 : SLOTS;
  double tot[SLOTS][NDOT];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
#pragma unroll
    for (int d = 0; d < NDOT; ++d) tot[j][d] = j < NS_ ? warp_sum(acc[j][d]) : 0.0;
#if NI_FILL_STATS
  const long long tw0 = clock64();
#endif
  while (fbt - vload_warp(&fb.head) >= FQ) __nanosleep(32);
#if NI_FILL_STATS
  if (lane == 0) NI_STAT(2, clock64() - tw0);
#endif
  FinishRec& r = fb.rec[fbt % FQ];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
#pragma unroll
    for (int d = 0; d < NDOT; ++d)
      if (lane == j * NDOT + d) r.sum[j][d] = tot[j][d];
  if (lane == 8) r.comp[0] = k.comp[0];
  if (lane == 9) r.comp[1] = k.comp[1];
  if (lane == 10) r.pbase = k.pbase;
  if (lane == 11) r.nslot = item_n_flags(k.flags);
  if (lane == 12) r.g = k.g;
  if (lane == 13) r.n = k.n;
  if (lane == 14) r.par = k.par;
  if (lane == 15) r.live = k.live;
  __syncwarp();
  ++fbt;
  if (lane == 0) {
    __threadfence_block();
    vstore(&fb.tail, fbt);
  }
}

// Initial live-item lists per group.
__device__ void initial_lists(const FillArgs& a, int gwarp, int nwarps) {
  const int lane = threadIdx.x & 31;
  for (int k = gwarp * 32 + lane; k < a.nitems; k += nwarps * 32) {
    if (!item_live(a, k)) continue;
    const int32_t g = a.cgrp[a.items[k].comp[0]];
    const int32_t pos = atomicAdd(a.gcnt + g, 1);
    a.active_items[a.gstart[g] + pos] = k;
  }
}

// A worker warp: take items from its mailbox and sweep them, streaming rows
// from one item into the next.
template <int CONN, bool EW>
__device__ void worker_loop(const FillArgs& a, unsigned char* ring, Mailbox& mb, FinishBox& fb,
                            const CtaShared& sh) {
  const int lane = threadIdx.x & 31;
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t vpitch = 16u * a.P;
  Issuer is;
  Cur cur;
  const Claim* nx = nullptr;
  int mbh = 0, fbt = 0;  // worker-owned counters (mailbox head, finish tail)
  bool have = false;
#if NI_FILL_STATS
  const long long t_start = clock64();
  long long t_idle = 0, n_items = 0;
#endif
  for (;;) {
    if (!have) {
      if (mbh == vload_warp(&mb.tail)) {
        if (vload_warp(&sh.done)) break;
#if NI_FILL_STATS
        const long long ti = clock64();
        __nanosleep(NI_IDLE_NS);
        t_idle += clock64() - ti + 40;
#else
        __nanosleep(NI_IDLE_NS);
#endif
        continue;
      }
      __threadfence_block();
      nx = &mb.slot[mbh % MB];
      have = true;
      issuer_start<EW>(a, nx->item, nx->par, is);
      for (int j = 0; j < LA; ++j) issue_row<EW>(ring_s, j, is, vpitch);
    }
    load_cur(*nx, cur);
    __syncwarp();
    ++mbh;
    if (lane == 0) vstore(&mb.head, mbh);
    bool has_next = false;
    if (cur.flags & 0x100)
      sweep_item<CONN, true, EW>(a, ring, mb, mbh, nx, is, cur, has_next, fb, fbt);
    else
      sweep_item<CONN, false, EW>(a, ring, mb, mbh, nx, is, cur, has_next, fb, fbt);
    if (!has_next) {
      cp_wait<0>();
      have = false;
    }
#if NI_FILL_STATS
    ++n_items;
#endif
  }
  cp_wait<0>();
#if NI_FILL_STATS
  if (lane == 0) {
    NI_STAT(0, clock64() - t_start);
    NI_STAT(1, t_idle);
    NI_STAT(3, n_items);
  }
#endif
}

// The whole CG of every component: one persistent cooperative launch.  A
// group's batch is one CG iteration of its components; the scheduler warp
// that retires the last item of a batch (after the per-component finalisers
// of all its items ran) publishes the group's next batch.  No grid-wide
// barrier per iteration: groups drift apart and every worker stays busy
// while any batch is open.
template <int CONN, int MINB, bool EW>
__global__ void __launch_bounds__(NT_FILL, MINB) fill_cg_kernel(const __grid_constant__ FillArgs a) {
  constexpr size_t kRing = ring_bytes<EW>();
  cg::grid_group grid = cg::this_grid();
  constexpr int WPC = NT_FILL / 32;
  const int gwarp = blockIdx.x * WPC + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * WPC;
  initial_lists(a, gwarp, nwarps);
  grid.sync();
  for (int g = blockIdx.x * NT_FILL + threadIdx.x; g < a.G; g += gridDim.x * NT_FILL) {
    const int32_t n = __ldcg(a.gcnt + g);
    if (n > 0) {
      atomicAdd(a.gactive, 1);
      // every group starts at parity 0 (v[0] holds b)
      if (a.window <= 0 || g < a.window) publish(a, g, 0, n);
    }
  }
  extern __shared__ __align__(16) unsigned char smem[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(smem + kRing * WORKERS);
  for (int i = threadIdx.x; i < int(sizeof(CtaShared) / sizeof(int)); i += NT_FILL)
    reinterpret_cast<int*>(&sh)[i] = 0;
  grid.sync();
  const int w = threadIdx.x >> 5;
  if (w == WORKERS) scheduler_loop(a, sh);
  else worker_loop<CONN, EW>(a, smem + kRing * w, sh.mb[w], sh.fb[w], sh);
}

// Initial ||b||^2 per component and the state of every component.  One warp
// per item, like the sweeps.
__global__ void __launch_bounds__(NT) init_norm_kernel(const __grid_constant__ FillArgs a, double rtol) {
  const int gwarp = blockIdx.x * WPB + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * WPB;
  const int lane = threadIdx.x & 31;
  for (int k = gwarp; k < a.nitems; k += nwarps) {
    const Item it = a.items[k];
    const int xr = it.x0 - 1 + lane;
    const bool on = lane >= 1 && lane <= SW && xr < a.W;
    double acc[SLOTS][NDOT];
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
#pragma unroll
      for (int d = 0; d < NDOT; ++d) acc[j][d] = 0.0;
    const int yend = it.y1;
    if (on) {
      for (int y = it.y0; y < yend; ++y) {
        const int64_t o = int64_t(y + RM) * a.P + xr + XM;
        const int s = slot_of(it, a.lab[o]);
        if (s < 0) continue;
        const double rv = a.v[0][o].x;
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
      }
    });
  }
}

// status ACTIVE only while the initial norm pass counts arrivals; its
// finaliser sets the real state and the active count.
__global__ void init_state_kernel(uint8_t* __restrict__ status, uint8_t* __restrict__ final_status,
                                  uint8_t* __restrict__ xbuf, int32_t* __restrict__ iters,
                                  int32_t* __restrict__ cap, double* __restrict__ rho,
                                  const int32_t* __restrict__ comp_size, int C, int cg_max_iters) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    status[c] = comp_size[c] >= 2 ? ST_ACTIVE : ST_IDLE;
    final_status[c] = ST_CONVERGED;
    xbuf[c] = 0;
    iters[c] = 0;
    const int n = comp_size[c];
    cap[c] = n > cg_max_iters ? n : cg_max_iters;
    rho[c] = 0.0;
  }
}

__global__ void output_kernel(const float4* __restrict__ v0, const float4* __restrict__ v1,
                              const int32_t* __restrict__ labels,
                              const int32_t* __restrict__ comp_size,
                              const uint8_t* __restrict__ xbuf, int W, int P, int64_t npix,
                              double* __restrict__ z) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t l = labels[i];
    double out = 0.0;
    if (l >= 0 && comp_size[l] >= 2) {
      const int64_t o = (i / W + RM) * P + i % W + XM;
      out = double((xbuf[l] ? v1 : v0)[o].w);
    }
    z[i] = out;
  }
}

__global__ void status_out_kernel(const uint8_t* __restrict__ status,
                                  const int32_t* __restrict__ iters, int C,
                                  const int32_t* __restrict__ comp_size,
                                  int32_t* __restrict__ iters_out,
                                  int32_t* __restrict__ status_out,
                                  unsigned long long* __restrict__ px_iters,
                                  int32_t* __restrict__ max_iters) {
  unsigned long long acc = 0;
  int mx = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int it = iters[c];
    iters_out[c] = it;
    status_out[c] = status[c] == ST_CAPPED ? 1 : 0;
    if (comp_size[c] >= 2) acc += (unsigned long long)comp_size[c] * (unsigned long long)it;
    mx = it > mx ? it : mx;
  }
  atomicAdd(px_iters, acc);
  atomicMax(max_iters, mx);
}

// ---- lockstep groups: components that share an item (union-find over the
// item pairs); only components with items get a group
__global__ void grp_init_kernel(int32_t* __restrict__ parent, int C) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    parent[c] = c;
}

__global__ void grp_union_kernel(const Item* __restrict__ items, int nitems,
                                 int32_t* __restrict__ parent) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nitems; k += gridDim.x * blockDim.x) {
    const Item it = items[k];
    if (item_n(it) == 2) uf_union(parent, it.comp[0], it.comp[1]);
  }
}

__global__ void grp_root_kernel(int32_t* __restrict__ parent,
                                const int32_t* __restrict__ comp_nparts, int C,
                                int32_t* __restrict__ isroot) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    const int32_t r = uf_find(parent, c);
    isroot[c] = r == c && comp_nparts[c] > 0;
  }
}

__global__ void grp_assign_kernel(const int32_t* __restrict__ parent,
                                  const int32_t* __restrict__ gid,
                                  const int32_t* __restrict__ comp_nparts, int C,
                                  int32_t* __restrict__ cgrp) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x)
    cgrp[c] = comp_nparts[c] > 0 ? gid[uf_find(const_cast<int32_t*>(parent), c)] : -1;
}

__global__ void grp_size_kernel(const Item* __restrict__ items, int nitems,
                                const int32_t* __restrict__ cgrp, int32_t* __restrict__ gsize) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nitems; k += gridDim.x * blockDim.x)
    atomicAdd(gsize + cgrp[items[k].comp[0]], 1);
}

// ------------------------------------------------------------ workspace

struct FillWs {
  float4 *v0, *v1, *cf;
  float* hw;
  uint8_t* imask;
  int32_t* lab_p;
  int32_t *slot_base, *nslots, *nitems_strip, *item_base, *strip_comps, *partial_comp,
      *partial_idx, *plist, *keys_sorted;
  Item* items;
  int32_t *comp_size, *comp_nparts, *comp_pstart, *comp_cnt, *iters, *cap, *total, *total_items,
      *active_items;
  int32_t *parent, *isroot, *gid, *cgrp, *gsize, *gstart, *gcnt, *gdone, *gchg, *gactive, *ngroups;
  unsigned long long *gtk, *ring;
  uint32_t *ring_tail, *ring_hint, *gseq;
  int32_t* gnext;
  uint32_t R;
  double *partial, *rho, *alpha, *beta, *tol;
  uint8_t *status, *final_status, *xbuf;
  unsigned long long* px_iters;
  int32_t* max_iters;
  void* sort_ws;
  size_t sort_bytes;
  void* scan_ws;
};

// Batch ring capacity: at most one open batch per group sits ahead of the
// hint, plus exhausted entries the hint has not passed yet.
static uint32_t ring_cap(int C) {
  uint32_t r = 8192;
  while (r < 4u * uint32_t(C + 1) + 8192u) r <<= 1;
  return r;
}

static int pitch_of(int W) { return (W + XM + 48 + 15) & ~15; }
static int64_t padded_len(int rows, int W) { return int64_t(rows + RM + RB) * pitch_of(W); }

static void carve_fill(Carver& c, FillWs& w, int64_t npix, int rows, int W, int nstrips, int C,
                       bool weighted) {
  const int64_t npad = padded_len(rows, W);
  // every partial slot owns >= 1 pixel
  const int64_t P = npix;
  const int64_t NI = nstrips + P + 1;  // items (one per strip component at most)
  w.v0 = c.take<float4>(npad);
  w.v1 = c.take<float4>(npad);
  w.hw = c.take<float>(weighted ? 1 : npad);
  w.cf = c.take<float4>(weighted ? npad : 1);
  w.imask = c.take<uint8_t>(npad);
  w.lab_p = c.take<int32_t>(npad);
  w.slot_base = c.take<int32_t>(nstrips + 1);
  w.nslots = c.take<int32_t>(nstrips + 1);
  w.nitems_strip = c.take<int32_t>(nstrips + 1);
  w.item_base = c.take<int32_t>(nstrips + 1);
  w.strip_comps = c.take<int32_t>(int64_t(nstrips) * SPX);
  w.items = c.take<Item>(NI);
  w.active_items = c.take<int32_t>(NI);
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
  w.xbuf = c.take<uint8_t>(C + 1);
  w.parent = c.take<int32_t>(C + 1);
  w.isroot = c.take<int32_t>(C + 1);
  w.gid = c.take<int32_t>(C + 1);
  w.cgrp = c.take<int32_t>(C + 1);
  w.gsize = c.take<int32_t>(C + 1);
  w.gstart = c.take<int32_t>(C + 1);
  w.gcnt = c.take<int32_t>(C + 1);
  w.gdone = c.take<int32_t>(C + 1);
  w.gchg = c.take<int32_t>(C + 1);
  w.gtk = c.take<unsigned long long>(C + 1);
  w.gseq = c.take<uint32_t>(C + 1);
  w.R = ring_cap(C);
  w.ring = c.take<unsigned long long>(w.R);
  w.ring_tail = c.take<uint32_t>(1);
  w.ring_hint = c.take<uint32_t>(1);
  w.gactive = c.take<int32_t>(1);
  w.gnext = c.take<int32_t>(1);
  w.ngroups = c.take<int32_t>(1);
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
  *nsy = B * div_up(H, SH);
}

extern "C" int ni_fill_workspace_size(int B, int H, int W, int connectivity, int count,
                                      int weighted, size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  const int64_t npix = int64_t(B) * H * W;
  int nsx, nsy;
  strip_grid(B, H, W, &nsx, &nsy);
  Sizer s;
  FillWs w;
  carve_fill(s, w, npix, B * H, W, nsx * nsy, count, weighted != 0);
  *bytes = s.used;
  return NI_OK;
}

extern "C" int ni_fill(const int32_t* labels, int count, const double* omega_a,
                       const double* omega_b, const double* gamma, const uint8_t* eflags,
                       const double* w_a, const double* w_b, int B, int H, int W,
                       int connectivity, int model, double cg_tol, int cg_max_iters,
                       double* z_out, int32_t* comp_iters, int32_t* comp_status, void* workspace,
                       size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(model == 0 || (model == 1 && connectivity == 4), "bad model/connectivity");
  NI_CHECK_ARG(cg_tol > 0, "cg_tol must be positive");
  NI_CHECK_ARG(count >= 0, "count must be non-negative");
  NI_CHECK_ARG((w_a == nullptr) == (w_b == nullptr), "w_a and w_b go together");
  const bool weighted = w_a != nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  const int rows = B * H;
  const int P = pitch_of(W);
  int nsx, nsy;
  strip_grid(B, H, W, &nsx, &nsy);
  const int nstrips = nsx * nsy;
  Carver cv(workspace, workspace_bytes);
  FillWs w;
  carve_fill(cv, w, npix, rows, W, nstrips, count, weighted);
  if (!cv.ok() || !workspace) {
    set_error("ni_fill: workspace too small (%zu < %zu)", workspace_bytes, cv.used);
    return NI_ERR_WORKSPACE;
  }
  const int blocks = int(std::min<int64_t>((npix + 255) / 256, int64_t(kSMs) * 16));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_size, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_nparts, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_cnt, 0, sizeof(int32_t) * (count + 1), s));
  {  // zero margins and buffers of the padded layout
    const size_t npad = size_t(padded_len(rows, W));
    NI_CUDA_TRY(cudaMemsetAsync(w.v0, 0, npad * sizeof(float4), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.v1, 0, npad * sizeof(float4), s));
    if (weighted) NI_CUDA_TRY(cudaMemsetAsync(w.cf, 0, npad * sizeof(float4), s));
    else NI_CUDA_TRY(cudaMemsetAsync(w.hw, 0, npad * sizeof(float), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.imask, 0, npad, s));
    NI_CUDA_TRY(cudaMemsetAsync(w.lab_p, 0xff, npad * sizeof(int32_t), s));
  }
#define NI_PREP(CONN, MODEL, EW)                                                               \
  NI_COUNT_LAUNCH(), prep_kernel<CONN, MODEL, EW><<<blocks, 256, 0, s>>>(                      \
                         labels, omega_a, omega_b, gamma, eflags, w_a, w_b, H, W, P, npix, w.hw, \
                         w.cf, w.imask, w.lab_p, w.v0, w.comp_size)
  if (weighted) {
    if (connectivity == 8) NI_PREP(8, 0, true);
    else if (model == 0) NI_PREP(4, 0, true);
    else NI_PREP(4, 1, true);
  } else {
    if (connectivity == 8) NI_PREP(8, 0, false);
    else if (model == 0) NI_PREP(4, 0, false);
    else NI_PREP(4, 1, false);
  }
#undef NI_PREP
  NI_LAUNCH_CHECK();
  // ---- static reduction plan: strips -> items -> partial slots
  NI_COUNT_LAUNCH(), strip_comps_kernel<<<nstrips, NT, 0, s>>>(
                         labels, w.comp_size, H, W, nsx, nsy / B, w.nslots, w.strip_comps);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(w.nslots, w.slot_base, nstrips, w.total, w.scan_ws, s));
  // Items pair up to SLOTS components of a strip; pairing couples those
  // components into one lockstep group.  With many maps the groups (about
  // one per map) overlap each other well and pairing saves re-reading mixed
  // strips; with few maps one group per component overlaps far better.
  const char* pe = NI_ENV_ONCE("NI_FILL_PAIR");
  const int per = pe ? (atoi(pe) > 1 ? SLOTS : 1) : (B >= kPairMaps ? SLOTS : 1);
  NI_COUNT_LAUNCH(), item_counts_kernel<<<div_up(nstrips, 256), 256, 0, s>>>(w.nslots, nstrips, per,
                                                                            w.nitems_strip);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(w.nitems_strip, w.item_base, nstrips, w.total_items, w.scan_ws, s));
  NI_COUNT_LAUNCH(), strip_items_kernel<<<div_up(nstrips, 128), 128, 0, s>>>(
                         w.nslots, w.slot_base, w.item_base, w.strip_comps, nstrips, nsx, nsy / B,
                         H, per, w.items, w.partial_comp, w.partial_idx, w.comp_nparts);
  NI_LAUNCH_CHECK();
  int32_t NP = 0, NIt = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&NP, w.total, sizeof(NP), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaMemcpyAsync(&NIt, w.total_items, sizeof(NIt), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  if (NP > 0) {
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= count) ++end_bit;
    size_t sb = w.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_ws, sb, w.partial_comp, w.keys_sorted,
                                                w.partial_idx, w.plist, NP, 0, end_bit, s));
  }
  NI_TRY(exclusive_scan_i32(w.comp_nparts, w.comp_pstart, count + 1, nullptr, w.scan_ws, s));
  // ---- lockstep groups and their item regions
  int32_t G = 0;
  if (count > 0) {
    const int cb = div_up(count, 256);
    NI_COUNT_LAUNCH(), grp_init_kernel<<<cb, 256, 0, s>>>(w.parent, count);
    NI_LAUNCH_CHECK();
    if (NIt > 0) {
      NI_COUNT_LAUNCH(), grp_union_kernel<<<div_up(NIt, 256), 256, 0, s>>>(w.items, NIt, w.parent);
      NI_LAUNCH_CHECK();
    }
    NI_COUNT_LAUNCH(), grp_root_kernel<<<cb, 256, 0, s>>>(w.parent, w.comp_nparts, count, w.isroot);
    NI_LAUNCH_CHECK();
    NI_TRY(exclusive_scan_i32(w.isroot, w.gid, count, w.ngroups, w.scan_ws, s));
    NI_COUNT_LAUNCH(), grp_assign_kernel<<<cb, 256, 0, s>>>(w.parent, w.gid, w.comp_nparts, count,
                                                           w.cgrp);
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemcpyAsync(&G, w.ngroups, sizeof(G), cudaMemcpyDeviceToHost, s));
    NI_CUDA_TRY(cudaStreamSynchronize(s));
  }
  NI_CUDA_TRY(cudaMemsetAsync(w.gsize, 0, sizeof(int32_t) * (G + 1), s));
  if (NIt > 0) {
    NI_COUNT_LAUNCH(), grp_size_kernel<<<div_up(NIt, 256), 256, 0, s>>>(w.items, NIt, w.cgrp,
                                                                       w.gsize);
    NI_LAUNCH_CHECK();
  }
  NI_TRY(exclusive_scan_i32(w.gsize, w.gstart, G + 1, nullptr, w.scan_ws, s));
  NI_CUDA_TRY(cudaMemsetAsync(w.gcnt, 0, sizeof(int32_t) * (G + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.gdone, 0, sizeof(int32_t) * (G + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.gchg, 0, sizeof(int32_t) * (G + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.gtk, 0, sizeof(unsigned long long) * (G + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.gseq, 0xff, sizeof(uint32_t) * (G + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.ring, 0xff, sizeof(unsigned long long) * w.R, s));
  NI_CUDA_TRY(cudaMemsetAsync(w.ring_tail, 0, sizeof(uint32_t), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.ring_hint, 0, sizeof(uint32_t), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.gactive, 0, sizeof(int32_t), s));
  const char* we = NI_ENV_ONCE("NI_FILL_WINDOW");
  const int window = we ? atoi(we) : 0;
  NI_CUDA_TRY(cudaMemcpyAsync(w.gnext, &window, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  FillArgs a;
  memset(&a, 0, sizeof(a));
  a.rows = rows;
  a.W = W;
  a.P = P;
  a.v[0] = w.v0;
  a.v[1] = w.v1;
  a.hw = w.hw;
  a.cf = w.cf;
  a.imask = w.imask;
  a.lab = w.lab_p;
  a.items = w.items;
  a.nitems = NIt;
  a.comp_pstart = w.comp_pstart;
  a.comp_plist = w.plist;
  a.comp_cnt = w.comp_cnt;
  a.partial = w.partial;
  a.G = G;
  a.cgrp = w.cgrp;
  a.gstart = w.gstart;
  a.active_items = w.active_items;
  a.gcnt = w.gcnt;
  a.gtk = w.gtk;
  a.gdone = w.gdone;
  a.gchg = w.gchg;
  a.ring = w.ring;
  a.R = w.R;
  a.ring_tail = w.ring_tail;
  a.ring_hint = w.ring_hint;
  a.gseq = w.gseq;
  a.gactive = w.gactive;
  a.window = window;
  // One queued item per worker keeps a few large components (single maps,
  // unpaired items) spread over more workers; with many lockstep groups two
  // queued items keep every worker's row stream continuous.
  {
    const char* me = NI_ENV_ONCE("NI_FILL_MB");
    a.mb = me ? atoi(me) : (per > 1 ? MB : 1);
    if (a.mb < 1) a.mb = 1;
    if (a.mb > MB) a.mb = MB;
  }
  a.gnext = w.gnext;
  a.rho = w.rho;
  a.alpha = w.alpha;
  a.beta = w.beta;
  a.tol = w.tol;
  a.iters = w.iters;
  a.cap = w.cap;
  a.status = w.status;
  a.final_status = w.final_status;
  a.xbuf = w.xbuf;
  if (count > 0) {
    NI_COUNT_LAUNCH(), init_state_kernel<<<div_up(count, 256), 256, 0, s>>>(
                           w.status, w.final_status, w.xbuf, w.iters, w.cap, w.rho, w.comp_size,
                           count, cg_max_iters);
    NI_LAUNCH_CHECK();
  }
  if (NIt > 0) {
    NI_COUNT_LAUNCH(), init_norm_kernel<<<div_up(NIt, WPB), NT, 0, s>>>(a, cg_tol);
    NI_LAUNCH_CHECK();
  }
  // ---- the whole CG: one persistent cooperative launch
  {
    void* kfn;
    if (weighted)
      kfn = connectivity == 8 ? (void*)fill_cg_kernel<8, 1, true> : (void*)fill_cg_kernel<4, 1, true>;
    else
      kfn = connectivity == 8 ? (void*)fill_cg_kernel<8, 1, false>
                              : (void*)fill_cg_kernel<4, 1, false>;
    const size_t kSmemBytes = weighted ? smem_bytes<true>() : smem_bytes<false>();
    int dev = 0, sms = 0, per_sm = 0;
    NI_CUDA_TRY(cudaGetDevice(&dev));
    NI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    NI_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kSmemBytes)));
    NI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NT_FILL, kSmemBytes));
    int G = per_sm * sms;
    const int need = div_up(NIt > 0 ? NIt : 1, WORKERS);
    if (G > need) G = need;
    if (G < 1) G = 1;
    void* args[] = {&a};
    cudaEvent_t e0, e1;
    NI_CUDA_TRY(cudaEventCreate(&e0));
    NI_CUDA_TRY(cudaEventCreate(&e1));
#if NI_FILL_STATS
    unsigned long long zst[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    NI_CUDA_TRY(cudaMemcpyToSymbolAsync(g_fill_stats, zst, sizeof(zst), 0, cudaMemcpyHostToDevice, s));
    {
      static int zn[kTraceG];
      NI_CUDA_TRY(cudaMemcpyToSymbolAsync(g_pub_n, zn, sizeof(zn), 0, cudaMemcpyHostToDevice, s));
    }
#endif
    NI_CUDA_TRY(cudaEventRecord(e0, s));
    NI_COUNT_LAUNCH();
    NI_CUDA_TRY(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(NT_FILL), args, kSmemBytes, s));
    NI_CUDA_TRY(cudaEventRecord(e1, s));
    g_fill_report.grid = G;
    g_fill_report.ntiles = NIt;
    g_fill_report.npartials = NP;
    NI_CUDA_TRY(cudaMemsetAsync(w.px_iters, 0, sizeof(unsigned long long), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.max_iters, 0, sizeof(int32_t), s));
    if (count > 0) {
      NI_COUNT_LAUNCH(), status_out_kernel<<<div_up(count, 256), 256, 0, s>>>(
                             w.status, w.iters, count, w.comp_size, comp_iters, comp_status,
                             w.px_iters, w.max_iters);
      NI_LAUNCH_CHECK();
    }
    NI_COUNT_LAUNCH(), output_kernel<<<blocks, 256, 0, s>>>(w.v0, w.v1, labels, w.comp_size,
                                                           w.xbuf, W, P, npix, z_out);
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
#if NI_FILL_STATS
    unsigned long long h[8];
    NI_CUDA_TRY(cudaMemcpyFromSymbol(h, g_fill_stats, sizeof(h)));
    fprintf(stderr,
            "fill stats: groups=%d worker idle=%.1f%% finish-wait=%.1f%% cycles/item=%.0f | "
            "scheduler retire=%.1f%% claim=%.1f%% items/claim=%.2f\n",
            a.G, 100.0 * h[1] / h[0], 100.0 * h[2] / h[0], double(h[0]) / double(h[3]),
            100.0 * h[5] / h[4], 100.0 * h[6] / h[4], double(h[3]) / double(h[7]));
    if (const char* tp = NI_ENV_ONCE("NI_FILL_TRACE")) {  // batch publish timeline per group
      static int hn[kTraceG];
      static unsigned long long ht[kTraceG * kTraceI];
      NI_CUDA_TRY(cudaMemcpyFromSymbol(hn, g_pub_n, sizeof(hn)));
      NI_CUDA_TRY(cudaMemcpyFromSymbol(ht, g_pub_trace, sizeof(ht)));
      FILE* f = fopen(tp, "w");
      if (f) {
        for (int g = 0; g < kTraceG && g < a.G; ++g)
          for (int i = 0; i < hn[g] && i < kTraceI; ++i)
            fprintf(f, "%d %d %llu %llu\n", g, i, ht[g * kTraceI + i] & ((1ull << 48) - 1),
                    ht[g * kTraceI + i] >> 48);
        fclose(f);
      }
    }
#endif
  }
  return NI_OK;
}

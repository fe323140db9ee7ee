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
// Data layout in HBM.  rows = B*H; pixel (y, x) lives at padded index
// (y + RM) * P + (x + XM) with zeroed margins, so no access needs a bounds
// check (RM = 2 rows top / RB rows bottom, XM = 16 columns left, >= 32
// right):
//   v[2]  : float4 {r, q, p, x} per pixel, double-buffered by iteration
//           parity (a sweep reads its neighbours' previous values while other
//           warps write the new ones): one 16-B load and one 16-B store per
//           pixel and iteration
//   hw    : float32 W_a = gamma_a^2 / 2  (c_ab = hw_a + hw_b)
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
// Work decomposition: strips of 30 columns x 30 rows.  A warp processes a
// strip ("item") by marching down its rows: raw rows are prefetched into a
// 6-row register ring four rows ahead, each row's p' = r + beta p is formed
// once and shuffled to the neighbouring lanes (lanes 0 and 31 hold the halo
// columns), and the row loop is unrolled by the ring period so no register
// moves wait on loads.  No block barrier anywhere in a sweep.  A strip
// touching several multi-pixel components becomes ceil(n/2) "mixed" items of
// <= 2 components that read labels; a strip with one component is a "pure"
// item (singleton / invalid pixels carry r = q = p = x = 0 and stay 0).
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
constexpr int SH = 30;     // strip height (centre rows per item)
constexpr int SPX = 1024;  // padded pixels per strip (sort buffer)
constexpr int NT = 256;    // threads per CTA (8 warps)
constexpr int WPB = NT / 32;
constexpr int SLOTS = 2;  // components per item
constexpr int NDOT = 4;   // <p,q>, <r,q>, <q,q>, <r,r>
constexpr int RING = 6;   // raw row ring (row L+4 is loaded at centre row L)
constexpr int XM = 16;    // left margin (columns)
constexpr int RM = 2;     // top margin (rows)
constexpr int RB = 34;    // bottom margin (rows): every item streams 32 rows

enum : uint8_t { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_CAPPED = 2, ST_IDLE = 3, ST_FLUSH = 4 };

// One work item: a strip and up to 2 of its components.
struct __align__(16) Item {
  int32_t x0, y0;  // top-left centre pixel of the strip (column of lane 1)
  int32_t pbase;   // first partial slot of this item
  int32_t flags;   // bits 0-7: components in the item (1..2); bit 8: pure strip
  int32_t comp[SLOTS];
  int32_t pad[2];
};

__device__ __forceinline__ int item_n(const Item& it) { return it.flags & 0xFF; }
__device__ __forceinline__ bool item_pure(const Item& it) { return (it.flags >> 8) & 1; }

struct FillArgs {
  int rows, W, P;
  long long* trace;  // optional: per iteration (globaltimer, active items)
  int trace_len;
  float4* v[2];
  const float* hw;
  const uint8_t* imask;
  const int32_t* lab;  // padded labels
  // plan
  const Item* items;
  int nitems;
  const int32_t* comp_pstart;  // [C+1] partial range per component
  const int32_t* comp_plist;   // [P] partial indices grouped by component
  int32_t* comp_cnt;           // [C] arrival counters (zero between sweeps)
  double* partial;             // [P][NDOT]
  int32_t* active_items;       // [2][nitems]
  int32_t* nactive_items;      // [2]
  int32_t* ticket;             // [2] dynamic item scheduling, by sweep parity
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
  int32_t* active;        // components still ACTIVE or FLUSH
  int32_t* changed;       // a component changed state during the last sweep
};

// ----------------------------------------------------------------- setup

// Padded-layout setup: v[0] = {b, 0, 0, 0}, hw, imask, labels.
template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) prep_kernel(
    const int32_t* __restrict__ labels, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int P, int64_t npix,
    float* __restrict__ hw, uint8_t* __restrict__ imask, int32_t* __restrict__ lab_p,
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
    atomicAdd(comp_size + lab, 1);
    const double wa = 0.5 * (gamma[i] * gamma[i]);
    hw[o] = float(wa);
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
    imask[o] = m;
    v0[o] = make_float4(float(b), 0.f, 0.f, 0.f);
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
      it.pad[0] = it.pad[1] = 0;
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

// ---- the per-warp row stream (cp.async into a shared-memory ring)
//
// Every item is a stream of 32 rows (local rows 0..31 = real rows y0-1 ..
// y0+30) of its 32 columns (real x0-1 .. x0+30).  A warp's items follow each
// other in one continuous stream; row s of the stream lives in ring slot
// s % NS and is copied NS-2 rows ahead of its use, so the next item's first
// rows are in flight while the current item finishes.  Copies are
// cp.async (LDGSTS): no registers are held by in-flight loads.
constexpr int NS = 8;     // ring slots per warp
constexpr int IROWS = 32;  // stream rows per item

struct RowSlot {
  float4 v[32];      // r, q, p, x of lanes 0..31
  float h[36];       // hw window from the 16-B aligned column at or before lane 0
  int32_t lab[36];   // labels (mixed items), same window
  uint8_t m[48];     // imask window from the 16-B aligned column at or before lane 0
};
constexpr size_t kSmemPerWarp = sizeof(RowSlot) * NS;
constexpr size_t kSmemBytes = kSmemPerWarp * WPB;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue the copies of local row `j` of item `it` into `slot` (one commit
// group per row, possibly empty, in every lane).
__device__ __forceinline__ void issue_row(const FillArgs& a, const float4* __restrict__ vin,
                                          const Item* it, int j, RowSlot& slot) {
  const int lane = threadIdx.x & 31;
  if (it) {
    const int c0 = it->x0 - 1 + XM;                      // padded column of lane 0
    const int64_t rowo = int64_t(it->y0 - 1 + j + RM) * a.P;
    cp_async16(&slot.v[lane], vin + rowo + c0 + lane);
    const int ah = c0 & ~3;  // 16-B aligned float window
    if (lane < 9) cp_async16(&slot.h[4 * lane], a.hw + rowo + ah + 4 * lane);
    if (!item_pure(*it) && lane < 9) cp_async16(&slot.lab[4 * lane], a.lab + rowo + ah + 4 * lane);
    const int am = c0 & ~15;  // 16-B aligned byte window
    if (lane < 3) cp_async16(&slot.m[16 * lane], a.imask + rowo + am + 16 * lane);
  }
  cp_commit();
}

// A row of the compute ring: r_k, p_k = r_k + beta p_{k-1}, x_k formed with
// the pixel's own component (only intra-component neighbours are ever read,
// and those share the centre's alpha and beta), plus the left / right
// neighbours' p' and hw (warp shuffles; lanes 0 / 31 are the halo).
struct Row {
  float pn, h, pl, pr, hl, hr, rn, xn;
  uint32_t m;  // imask | (slot + 1) << 8
};

template <bool PURE>
__device__ __forceinline__ Row derive(const RowSlot& sl, const Item& it, const Coefs& k) {
  const int lane = threadIdx.x & 31;
  const int c0 = it.x0 - 1 + XM;
  const int dh = c0 & 3, dm = c0 & 15;
  const float4 v = sl.v[lane];
  float al = k.al[0], be = k.be[0];
  int s = 0;
  if (!PURE) {
    s = slot_of(it, sl.lab[dh + lane]);
    al = 0.f;
    be = 0.f;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
      if (j == s) {
        al = k.al[j];
        be = k.be[j];
      }
  }
  Row o;
  o.rn = fmaf(-al, v.y, v.x);
  o.pn = fmaf(be, v.z, o.rn);
  o.xn = fmaf(al, v.z, v.w);
  o.h = sl.h[dh + lane];
  o.m = uint32_t(sl.m[dm + lane]) | (uint32_t(s + 1) << 8);
  o.pl = __shfl_up_sync(0xffffffffu, o.pn, 1);
  o.pr = __shfl_down_sync(0xffffffffu, o.pn, 1);
  o.hl = __shfl_up_sync(0xffffffffu, o.h, 1);
  o.hr = __shfl_down_sync(0xffffffffu, o.h, 1);
  return o;
}

struct Stream {
  RowSlot* ring;  // NS slots of this warp
  uint32_t pos;   // stream row of the current item's local row 0
};

// One CG sweep over one item (see the header).  On entry the stream holds
// this item's rows 0..NS-3 (issued); `nxt` is the following item (or null)
// whose first rows are issued as this item's rows run out.
template <int CONN, bool PURE>
__device__ __forceinline__ void sweep_item(const FillArgs& a, Stream& st, const Item& it,
                                           const Coefs& k, int par, const Item* nxt) {
  const int lane = threadIdx.x & 31;
  const int xr = it.x0 - 1 + lane;  // real column of this lane
  const bool center_lane = lane >= 1 && lane <= SW && xr < a.W;
  const float4* __restrict__ vin = a.v[par];
  float4* __restrict__ vout = a.v[par ^ 1];
  double acc[SLOTS][NDOT];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j)
#pragma unroll
    for (int d = 0; d < NDOT; ++d) acc[j][d] = 0.0;
  const int nrows = min(SH, a.rows - it.y0);  // centre rows (local rows 1..nrows)
  const int64_t o0 = int64_t(it.y0 - 1 + RM) * a.P + (xr + XM);
  const int64_t P = a.P;
  // top up: rows NS-2 and NS-1... so that rows 0..NS-2 are issued here
  // (the previous item issued this item's rows 0..NS-4)
  auto issue_local = [&](int j) {  // local row j of this item or of the next
    const uint32_t sp = st.pos + j;
    if (j < IROWS) issue_row(a, vin, &it, j, st.ring[sp % NS]);
    else issue_row(a, vin, nxt, j - IROWS, st.ring[sp % NS]);
  };
  issue_local(NS - 3);
  issue_local(NS - 2);
  // rows 0 and 1 are complete once at most NS-3 younger groups are pending
  cp_wait<NS - 3>();
  __syncwarp();
  Row der[3];
  der[0] = derive<PURE>(st.ring[(st.pos + 0) % NS], it, k);
  der[1] = derive<PURE>(st.ring[(st.pos + 1) % NS], it, k);
  for (int g = 0; g < SH; g += 3) {
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int L = g + u + 1;  // centre local row
      // keep NS-2 rows ahead: row L+NS-2 (of this item or the next)
      issue_local(L + NS - 2);
      cp_wait<NS - 3>();  // row L+1 has landed
      __syncwarp();
      der[(u + 2) % 3] = derive<PURE>(st.ring[(st.pos + L + 1) % NS], it, k);
      const Row& U = der[u % 3];
      const Row& C = der[(u + 1) % 3];
      const Row& D = der[(u + 2) % 3];
      if (L > nrows) continue;
      const float pa = C.pn, ha = C.h;
      const uint32_t m = C.m;
      float q = 0.f;
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
      const int s = PURE ? 0 : int(m >> 8) - 1;  // -1: pixel not in this item
      uint8_t stt = ST_IDLE;
      if (PURE) {
        stt = k.st[0];
      } else {
#pragma unroll
        for (int j = 0; j < SLOTS; ++j)
          if (j == s) stt = k.st[j];
      }
      if (center_lane && (m & 0xFFu) != 0 && (stt == ST_ACTIVE || stt == ST_FLUSH)) {
        vout[o0 + int64_t(L) * P] = make_float4(C.rn, q, pa, C.xn);
        if (stt == ST_ACTIVE) {
          const double dp = pa, dq = q, dr = C.rn;
#pragma unroll
          for (int j = 0; j < SLOTS; ++j)
            if (j == s) {
              acc[j][0] = fma(dp, dq, acc[j][0]);
              acc[j][1] = fma(dr, dq, acc[j][1]);
              acc[j][2] = fma(dq, dq, acc[j][2]);
              acc[j][3] = fma(dr, dr, acc[j][3]);
            }
        }
      }
    }
  }
  st.pos += IROWS;
  bool live[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) live[j] = k.st[j] == ST_ACTIVE || k.st[j] == ST_FLUSH;
  item_finish(a, it, acc, live, [&](int32_t c, const double* d) {
    if (__ldcg(a.status + c) == ST_FLUSH) {  // the pending update is applied
      a.status[c] = __ldcg(a.final_status + c);
      a.xbuf[c] = uint8_t(par ^ 1);
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

__device__ __forceinline__ int draw_ticket(const FillArgs& a, int par) {
  int k = 0;
  if ((threadIdx.x & 31) == 0) k = atomicAdd(a.ticket + par, 1);
  return __shfl_sync(0xffffffffu, k, 0);
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
    a.ticket[0] = 0;
    a.ticket[1] = 0;
  }
  grid.sync();
  rebuild_items(a, 0, gwarp, nwarps);
  grid.sync();
  for (int it = 0;; ++it) {
    if (__ldcg(a.active) == 0) break;
    const int par = it & 1;
    // the other parity's ticket was last used by the previous sweep (done)
    if (blockIdx.x == 0 && threadIdx.x == 0) a.ticket[par ^ 1] = 0;
    const int n = __ldcg(a.nactive_items + cur);
    if (a.trace && it < a.trace_len && blockIdx.x == 0 && threadIdx.x == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[2 * it] = t;
      a.trace[2 * it + 1] = n;
    }
    // dynamic item scheduling: tickets are drawn one item ahead; the row
    // stream runs straight from one item into the next
    extern __shared__ __align__(16) unsigned char smem[];
    Stream st;
    st.ring = reinterpret_cast<RowSlot*>(smem + kSmemPerWarp * (threadIdx.x >> 5));
    st.pos = 0;
    int k = draw_ticket(a, par);
    Item item, nitem;
    Coefs kc, kn;
    bool has = k < n;
    if (has) {
      item = a.items[__ldcg(a.active_items + cur * a.nitems + k)];
      item_coefs(a, item, kc);
      for (int j = 0; j < NS - 3; ++j)
        issue_row(a, a.v[par], &item, j, st.ring[j % NS]);
    }
    while (has) {
      const int nk = draw_ticket(a, par);
      const bool has_next = nk < n;
      if (has_next) {
        nitem = a.items[__ldcg(a.active_items + cur * a.nitems + nk)];
        item_coefs(a, nitem, kn);
      }
      if (item_pure(item)) sweep_item<CONN, true>(a, st, item, kc, par, has_next ? &nitem : nullptr);
      else sweep_item<CONN, false>(a, st, item, kc, par, has_next ? &nitem : nullptr);
      item = nitem;
      kc = kn;
      has = has_next;
    }
    cp_wait<0>();
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
    const int xr = it.x0 - 1 + lane;
    const bool on = lane >= 1 && lane <= SW && xr < a.W;
    double acc[SLOTS][NDOT];
#pragma unroll
    for (int j = 0; j < SLOTS; ++j)
#pragma unroll
      for (int d = 0; d < NDOT; ++d) acc[j][d] = 0.0;
    const int yend = min(it.y0 + SH, a.rows);
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
        atomicAdd(a.active, 1);
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

// ------------------------------------------------------------ workspace

struct FillWs {
  float4 *v0, *v1;
  float* hw;
  uint8_t* imask;
  int32_t* lab_p;
  int32_t *slot_base, *nslots, *nitems_strip, *item_base, *strip_comps, *partial_comp,
      *partial_idx, *plist, *keys_sorted;
  Item* items;
  int32_t *comp_size, *comp_nparts, *comp_pstart, *comp_cnt, *iters, *cap, *active, *changed,
      *total, *total_items, *active_items, *nactive_items, *ticket;
  double *partial, *rho, *alpha, *beta, *tol;
  uint8_t *status, *final_status, *xbuf;
  unsigned long long* px_iters;
  int32_t* max_iters;
  void* sort_ws;
  size_t sort_bytes;
  void* scan_ws;
};

static int pitch_of(int W) { return (W + XM + 48 + 15) & ~15; }
static int64_t padded_len(int rows, int W) { return int64_t(rows + RM + RB) * pitch_of(W); }

static void carve_fill(Carver& c, FillWs& w, int64_t npix, int rows, int W, int nstrips, int C) {
  const int64_t npad = padded_len(rows, W);
  // every partial slot owns >= 1 pixel
  const int64_t P = npix;
  const int64_t NI = nstrips + P / SLOTS + 1;  // items
  w.v0 = c.take<float4>(npad);
  w.v1 = c.take<float4>(npad);
  w.hw = c.take<float>(npad);
  w.imask = c.take<uint8_t>(npad);
  w.lab_p = c.take<int32_t>(npad);
  w.slot_base = c.take<int32_t>(nstrips + 1);
  w.nslots = c.take<int32_t>(nstrips + 1);
  w.nitems_strip = c.take<int32_t>(nstrips + 1);
  w.item_base = c.take<int32_t>(nstrips + 1);
  w.strip_comps = c.take<int32_t>(int64_t(nstrips) * SPX);
  w.items = c.take<Item>(NI);
  w.active_items = c.take<int32_t>(2 * NI);
  w.nactive_items = c.take<int32_t>(2);
  w.ticket = c.take<int32_t>(2);
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
  carve_fill(s, w, npix, B * H, W, nsx * nsy, count);
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
  const int P = pitch_of(W);
  int nsx, nsy;
  strip_grid(B, H, W, &nsx, &nsy);
  const int nstrips = nsx * nsy;
  Carver cv(workspace, workspace_bytes);
  FillWs w;
  carve_fill(cv, w, npix, rows, W, nstrips, count);
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
  {  // zero margins and buffers of the padded layout
    const size_t npad = size_t(padded_len(rows, W));
    NI_CUDA_TRY(cudaMemsetAsync(w.v0, 0, npad * sizeof(float4), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.v1, 0, npad * sizeof(float4), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.hw, 0, npad * sizeof(float), s));
    NI_CUDA_TRY(cudaMemsetAsync(w.imask, 0, npad, s));
    NI_CUDA_TRY(cudaMemsetAsync(w.lab_p, 0xff, npad * sizeof(int32_t), s));
  }
#define NI_PREP(CONN, MODEL)                                                                   \
  NI_COUNT_LAUNCH(), prep_kernel<CONN, MODEL><<<blocks, 256, 0, s>>>(                          \
                         labels, omega_a, omega_b, gamma, eflags, H, W, P, npix, w.hw, w.imask, \
                         w.lab_p, w.v0, w.comp_size)
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
  FillArgs a;
  memset(&a, 0, sizeof(a));
  static long long* trace_buf = nullptr;
  if (getenv("NI_FILL_TRACE")) {  // debug: per-iteration timeline
    if (!trace_buf) NI_CUDA_TRY(cudaMalloc(&trace_buf, sizeof(long long) * 2 * 65536));
    NI_CUDA_TRY(cudaMemsetAsync(trace_buf, 0, sizeof(long long) * 2 * 65536, s));
    a.trace = trace_buf;
    a.trace_len = 65536;
  }
  a.rows = rows;
  a.W = W;
  a.P = P;
  a.v[0] = w.v0;
  a.v[1] = w.v1;
  a.hw = w.hw;
  a.imask = w.imask;
  a.lab = w.lab_p;
  a.items = w.items;
  a.nitems = NIt;
  a.comp_pstart = w.comp_pstart;
  a.comp_plist = w.plist;
  a.comp_cnt = w.comp_cnt;
  a.partial = w.partial;
  a.active_items = w.active_items;
  a.nactive_items = w.nactive_items;
  a.ticket = w.ticket;
  a.rho = w.rho;
  a.alpha = w.alpha;
  a.beta = w.beta;
  a.tol = w.tol;
  a.iters = w.iters;
  a.cap = w.cap;
  a.status = w.status;
  a.final_status = w.final_status;
  a.xbuf = w.xbuf;
  a.active = w.active;
  a.changed = w.changed;
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
    // register budget variant (NI_FILL_MINB = CTAs/SM it is sized for)
    const char* mb = getenv("NI_FILL_MINB");
    const int minb = mb ? atoi(mb) : 2;
    void* kfn;
    if (connectivity == 8)
      kfn = minb == 3 ? (void*)fill_cg_kernel<8, 3> : (void*)fill_cg_kernel<8, 2>;
    else
      kfn = minb == 3 ? (void*)fill_cg_kernel<4, 3> : (void*)fill_cg_kernel<4, 2>;
    int dev = 0, sms = 0, per_sm = 0;
    NI_CUDA_TRY(cudaGetDevice(&dev));
    NI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    NI_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kSmemBytes)));
    NI_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NT, kSmemBytes));
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
    NI_CUDA_TRY(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(NT), args, kSmemBytes, s));
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
    if (a.trace) {  // debug trace dump (NI_FILL_TRACE=path)
      static long long host[2 * 65536];
      NI_CUDA_TRY(cudaMemcpy(host, a.trace, sizeof(host), cudaMemcpyDeviceToHost));
      FILE* f = fopen(getenv("NI_FILL_TRACE"), "w");
      if (f) {
        for (int k = 0; k < 65536 && host[2 * k]; ++k)
          fprintf(f, "%lld %lld\n", host[2 * k], host[2 * k + 1]);
        fclose(f);
      }
    }
  }
  return NI_OK;
}

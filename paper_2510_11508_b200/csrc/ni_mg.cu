// K3 -- fill_components (solver.py:195-239) as ONE batched,
// multigrid-preconditioned conjugate-gradient solve over every component of
// every map of the batch.
//
// What the reference computes.  Per component c, scipy's CG on the normal
// equations (A^T W A) x = A^T W b from x0 = 0, stopped when ||r|| <
// rtol ||b|| (cap max(cg_max_iters, n_c); solver.py:97-122).  At the fill
// state z = 0 every bilateral factor is 1/2 (continuity.py:302-308), so
// A^T W A is the graph Laplacian of the component's valid edges with
// conductance c_ab = gamma_a^2/2 + gamma_b^2/2.  CG
// from 0 keeps x in range(A): the solution is mean-free on every connected
// part of the positive-conductance graph (a "solve unit"; a component is one
// unit unless degenerate edges split it).
//
// What this file computes.  The same systems solved to the same relative
// residual (per unit ||r_u|| < rtol ||b_u||, which implies the component's
// ||r_c|| < rtol ||b_c||), with the fewest passes over HBM: CG preconditioned
// by one V-cycle of a component-aware aggregation multigrid, then the
// null-space component removed per unit (the unpreconditioned CG's gauge).
// A tightly converged solve stays within ~1e-7 of scipy's iterate, five
// orders of magnitude inside the parity bound (scripts/
// solver_tolerance_study.py); the CG needs ~1,000-2,600 sweeps per component
// of a 1024^2 map, the MG-PCG 9-14 V-cycles.
//
// Hierarchy (built once per call, all maps at once).  Level 0 is the pixel
// grid.  A level-l unknown is a (2^l x 2^l block, unit) aggregate: the
// pixels of one unit inside one block, so aggregates never mix units and the
// preconditioner is block-diagonal over units.  Unknowns are sorted by
// (map, block row, block column, unit) and found through a per-level block
// table; each has 8 neighbour links (same unit in the 8 adjacent blocks),
// Galerkin conductances (fixed-order sums of the finer links crossing the
// two aggregates: P^T A P of the piecewise-constant prolongation), its
// parent and (l >= 2) up to 4 children.  Coarsening stops when no link is
// left (every unit is one aggregate).
//
// V-cycle (symmetric, so plain PCG applies): damped Jacobi from zero
// (omega = 0.8), residual, restriction (sum over children), recursion,
// prolongation scaled by 2.0 (over-correction, the standard fix for
// piecewise-constant prolongation), damped-Jacobi post-smoothing; one sweep
// before and after the coarse correction on levels 0 and 1, two on the
// (cheap) levels >= 2; the levels below ~8,000 unknowns run in one
// single-CTA launch (tail_kernel).
//
// PCG in the Chronopoulos-Gear form: one fine "down" pass (vector updates
// p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s fused with the
// pre-smoothing, residual and restriction of the new r) and one fine "up"
// pass (prolongation, post-smoothing -> u = M r, w = A u and the three dot
// products (r,u), (w,u), (r,r) per unit) per iteration, so each iteration
// has exactly one reduction point.  The stop test is scipy's, evaluated on
// the recursive residual at the top of the iteration.
//
// Fine-level planes (padded: pixel (y, x) of the stacked B*H rows at
// (y + RM) * P + x + XM, zero margins): x, r, p, s, u, w (f32), hw =
// gamma^2/2 (f32), dinv (f32), imask (u8: bit k = forward edge k, bit 4+k =
// backward edge k, set iff intra-component, valid and c > 0), par0 (i32:
// the level-1 aggregate), slot (u16: index of the pixel's unit in its
// tile's unit list).  Tiles of 64 x 32 pixels never straddle two maps; a CTA
// stages a tile plus a 1- or 2-pixel halo of the planes it stencils in
// shared memory.
//
// Reductions are deterministic: per (tile, unit) slot a fixed-order f64 sum,
// per unit its slots in slot order (a stable radix sort gives the order).
// Coarse conductances, restrictions and counts are fixed-order gathers.  No
// floating-point atomics: reruns are bit-identical.
#include <stdlib.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cub/device/device_radix_sort.cuh>
#include <cuda_bf16.h>

#include "ni_common.cuh"

namespace ni {
namespace mg {

constexpr int TX = 64;  // tile width (pixels)
constexpr int TY = 32;  // tile height
constexpr int TPX = TX * TY;
constexpr int NT = 256;  // threads per tile CTA: 2 x 2-pixel blocks each
constexpr int XM = 16;   // left / right margin (columns)
constexpr int RM = 2;    // top margin (rows)
constexpr int RB = TY + 4;  // bottom margin (rows)
constexpr int MAXLEV = 24;
constexpr uint16_t NOSLOT = 0xFFFF;
constexpr int NPART = 6;  // per-slot partials: (r,u) (w,u) (r,r) sum u, sum r, sum w
#ifndef NI_MG_OMEGA
#define NI_MG_OMEGA 0.8f
#endif
#ifndef NI_MG_OC
#define NI_MG_OC 2.0f  // with two sweeps on levels >= 2 (blueprint, three C5 maps: 1.9 9.0-9.4
#endif                 // iterations per pixel, 2.0 8.2-8.5, 2.1 9.5; GPU C5 step 51.8 -> 50.0 ms)
constexpr float OM = NI_MG_OMEGA;  // damped-Jacobi weight
constexpr float OC = NI_MG_OC;     // coarse-correction scale

enum : uint8_t { U_ACTIVE = 0, U_CONV = 1, U_CAPPED = 2, U_IDLE = 3 };

struct Geo {
  int B, H, W, P, nTX, nTY, ntiles, rows;
  int64_t npix, npad;
};

static Geo make_geo(int B, int H, int W) {
  Geo g;
  g.B = B;
  g.H = H;
  g.W = W;
  g.nTX = div_up(W, TX);
  g.nTY = div_up(H, TY);
  g.P = g.nTX * TX + 2 * XM;
  g.ntiles = B * g.nTX * g.nTY;
  g.rows = B * H;
  g.npix = int64_t(B) * H * W;
  g.npad = int64_t(g.rows + RM + RB) * g.P;
  return g;
}

__host__ __device__ __forceinline__ int64_t pidx(int P, int y, int x) {
  return int64_t(y + RM) * P + x + XM;
}

// direction of a neighbouring block (dx, dy in -1..1, not both 0) -> 0..7;
// opposite(d) = 7 - d
__host__ __device__ __forceinline__ int dir_of(int dx, int dy) {
  const int i = (dy + 1) * 3 + (dx + 1);
  return i < 4 ? i : i - 1;
}
__host__ __device__ __forceinline__ int dir_dx(int d) {
  const int i = d < 4 ? d : d + 1;
  return i % 3 - 1;
}
__host__ __device__ __forceinline__ int dir_dy(int d) {
  const int i = d < 4 ? d : d + 1;
  return i / 3 - 1;
}

// W_a = gamma_a^2 / 2 at the fill state (continuity.py:302-308), as stored
__device__ __forceinline__ float hw_of(double g) { return float(0.5 * (g * g)); }

struct Tile {
  int m, y0, y1, x0, x1;
};

__device__ __forceinline__ Tile tile_of(int t, int H, int W, int nTX, int nTY) {
  Tile T;
  const int per = nTX * nTY;
  T.m = t / per;
  const int r = t - T.m * per;
  const int ty = r / nTX, tx = r - ty * nTX;
  T.y0 = T.m * H + ty * TY;
  T.y1 = min(T.y0 + TY, (T.m + 1) * H);
  T.x0 = tx * TX;
  T.x1 = min(T.x0 + TX, W);
  return T;
}

// ------------------------------------------------------------ fine setup

// hw, b (into r), imask per pixel; component sizes; count of same-label
// edges that carry no conductance (then units != components).  2-D launch
// (x: column, y: stacked row); every neighbour's label / gamma / flags is
// loaded before any is compared, so the 2 x KF gathers of a pixel are in
// flight together instead of in dependent chains.
template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) prep_kernel(
    const int32_t* __restrict__ labels, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int P, int64_t npix,
    float* __restrict__ hw, float* __restrict__ rvec, uint8_t* __restrict__ imask,
    float* __restrict__ dinv, int32_t* __restrict__ comp_size, int32_t* __restrict__ missing) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  const int u = blockIdx.x * 32 + (threadIdx.x & 31);
  const int row = blockIdx.y * 8 + (threadIdx.x >> 5);
  const bool in = u < W && int64_t(row) * W < npix;
  const int64_t i = int64_t(row) * W + u;
  const int32_t lab = in ? labels[i] : -1;
  int miss = 0;
  {
    const unsigned peers = __match_any_sync(0xffffffffu, lab);
    if (lab >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(comp_size + lab, __popc(peers));
  }
  if (lab >= 0) {
    const int vloc = row % H;
    const int64_t o = pidx(P, row, u);
    const uint8_t ef = eflags[i];
    const double gs = gamma[i];
    // forward (k) and backward (4 + k) neighbours: existence, then all loads
    bool fex[KF], bex[KF];
    int32_t fl[KF], bl[KF];
    double fg[KF], bg[KF], fo[KF], bo[KF], fob[KF], bob[KF];
    uint8_t bef[KF];
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
      fex[k] = (ef >> k) & 1;
      const int64_t jf = fex[k] ? i + int64_t(dv) * W + du : i;
      fl[k] = labels[jf];
      fg[k] = gamma[jf];
      fo[k] = omega_a[k * npix + i];
      fob[k] = MODEL == 0 ? 0.0 : omega_b[k * npix + i];
      const int uj = u - du, vj = vloc - dv;
      bex[k] = uj >= 0 && uj < W && vj >= 0;
      const int64_t jb = bex[k] ? i - int64_t(dv) * W - du : i;
      bl[k] = labels[jb];
      bg[k] = gamma[jb];
      bef[k] = eflags[jb];
      bo[k] = omega_a[k * npix + jb];
      bob[k] = MODEL == 0 ? 0.0 : omega_b[k * npix + jb];
    }
    const double wself = 0.5 * (gs * gs);
    const float hself = hw_of(gs);
    hw[o] = hself;
    uint8_t m = 0;
    double b = 0.0;
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      if (fex[k] && fl[k] == lab) {  // forward edge i -> j inside the component
        const bool ok = ((ef >> (4 + k)) & 1) && (hself + hw_of(fg[k])) > 0.f;
        if (ok) {
          m |= uint8_t(1u << k);
          const double wb = 0.5 * (fg[k] * fg[k]);
          const double oa = fo[k];
          const double ob = MODEL == 0 ? -oa : fob[k];
          b += wself * oa - wb * ob;  // A^T W b of rows 2e, 2e+1 (solver.py:83-93)
        } else {
          ++miss;
        }
      }
      if (bex[k] && ((bef[k] >> k) & 1) && bl[k] == lab && ((bef[k] >> (4 + k)) & 1) &&
          (hself + hw_of(bg[k])) > 0.f) {  // backward edge j -> i
        m |= uint8_t(1u << (4 + k));
        const double wj = 0.5 * (bg[k] * bg[k]);
        const double oa = bo[k];
        const double ob = MODEL == 0 ? -oa : bob[k];
        b += wself * ob - wj * oa;
      }
    }
    imask[o] = m;
    rvec[o] = float(b);
    // the Jacobi diagonal sum of c_ab over the stencil edges, in the order
    // the fine passes' stencil visits them (forward k, then backward k)
    if (m) {
      float d = 0.f;
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        if ((m >> k) & 1) d += hself + hw_of(fg[k]);
        if ((m >> (4 + k)) & 1) d += hself + hw_of(bg[k]);
      }
      dinv[o] = 1.0f / d;
    }
  }
  if (miss) atomicAdd(missing, miss);
}

// neighbour offset of imask bit `bit` in a row-major array of pitch S
template <int CONN>
__device__ __forceinline__ int nb_off(int bit, int S) {
  const int k = bit & 3;
  const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
  return bit < 4 ? dv * S + du : -(dv * S + du);
}

// ---- solve units.  Fast path (every same-label edge carries conductance):
// units are the components.  General path: union-find over the imask graph.
__global__ void unit_from_label_kernel(const int32_t* __restrict__ labels, int H, int W, int P,
                                       int64_t npix, const uint8_t* __restrict__ imask,
                                       int32_t* __restrict__ unit) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = pidx(P, int(uint32_t(i) / uint32_t(W)), int(uint32_t(i) % uint32_t(W)));
    if (imask[o]) unit[o] = labels[i];
  }
}

__global__ void cc_init_kernel(int W, int P, int64_t npix, const uint8_t* __restrict__ imask,
                               int32_t* __restrict__ parent) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x)
    parent[i] = imask[pidx(P, int(uint32_t(i) / uint32_t(W)), int(uint32_t(i) % uint32_t(W)))] ? int32_t(i) : -1;
}

template <int CONN>
__global__ void cc_union_kernel(int W, int P, int64_t npix, const uint8_t* __restrict__ imask,
                                int32_t* __restrict__ parent) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t m = imask[pidx(P, int(uint32_t(i) / uint32_t(W)), int(uint32_t(i) % uint32_t(W)))];
#pragma unroll
    for (int k = 0; k < KF; ++k)
      if ((m >> k) & 1)
        uf_union(parent, int32_t(i), int32_t(i + int64_t(fwd_dv(CONN, k)) * W + fwd_du(CONN, k)));
  }
}

__global__ void cc_flatten_kernel(int64_t npix, int32_t* __restrict__ parent,
                                  int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    int32_t r = parent[i];
    if (r >= 0) {
      r = uf_find(parent, int32_t(i));
      parent[i] = r;
    }
    flag[i] = r == int32_t(i);
  }
}

__global__ void cc_label_kernel(const int32_t* __restrict__ labels, int W, int P, int64_t npix,
                                const int32_t* __restrict__ parent,
                                const int32_t* __restrict__ rank, int32_t* __restrict__ unit,
                                int32_t* __restrict__ unit_comp) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = parent[i];
    if (r < 0) continue;
    unit[pidx(P, int(uint32_t(i) / uint32_t(W)), int(uint32_t(i) % uint32_t(W)))] = rank[r];
    if (r == int32_t(i)) unit_comp[rank[r]] = labels[i];
  }
}

__global__ void iota_kernel(int32_t* __restrict__ a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

// ---- block-wide helpers (NT threads)

// exclusive scan of one int per thread; returns the total in every thread
__device__ __forceinline__ int block_excl_scan(int v, int* sw, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();
  if (lane == 31) sw[wid] = inc;
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    const int s = sw[w];
    if (w < wid) base += s;
    tot += s;
  }
  total = tot;
  return base + inc - v;
}

// ---- tile plan: per tile the sorted distinct units (its slots), per pixel
// its slot
__global__ void __launch_bounds__(NT) plan_tile_kernel(int H, int W, int P, int nTX, int nTY,
                                                       const int32_t* __restrict__ unit,
                                                       uint16_t* __restrict__ slot,
                                                       int32_t* __restrict__ nslots,
                                                       int32_t* __restrict__ tmp) {
  __shared__ int32_t key[TPX];
  __shared__ int sw[NT / 32];
  const int t = blockIdx.x;
  const Tile T = tile_of(t, H, W, nTX, nTY);
  for (int e = threadIdx.x; e < TPX; e += NT) {
    const int y = T.y0 + e / TX, x = T.x0 + e % TX;
    int32_t k = INT32_MAX;
    if (y < T.y1 && x < T.x1) {
      const int32_t u = unit[pidx(P, y, x)];
      if (u >= 0) k = u;
    }
    key[e] = k;
  }
  // fast path: a tile holding at most one unit (most tiles) needs no sort
  {
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (int e = threadIdx.x; e < TPX; e += NT) {
      const int32_t k = key[e];
      if (k != INT32_MAX) {
        lo = min(lo, k);
        hi = max(hi, k);
      }
    }
    __shared__ int32_t s_lo, s_hi;
    if (threadIdx.x == 0) {
      s_lo = INT32_MAX;
      s_hi = INT32_MIN;
    }
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&s_lo, lo);
      atomicMax(&s_hi, hi);
    }
    __syncthreads();
    lo = s_lo;
    hi = s_hi;
    if (lo == INT32_MAX || lo == hi) {
      const int total = lo == INT32_MAX ? 0 : 1;
      if (threadIdx.x == 0) {
        nslots[t] = total;
        if (total) tmp[int64_t(t) * TPX] = lo;
      }
      if (total)
        for (int e = threadIdx.x; e < TPX; e += NT)
          if (key[e] != INT32_MAX) slot[pidx(P, T.y0 + e / TX, T.x0 + e % TX)] = 0;
      return;
    }
    // a few units: extract them in ascending order by repeated block minima
    // (one pass over the tile each) instead of sorting the whole tile
    constexpr int kQuick = 16;
    __shared__ int32_t s_units[kQuick];
    __shared__ int32_t s_next;
    int total = 1;
    int32_t prev = lo;
    if (threadIdx.x == 0) s_units[0] = lo;
    while (total <= kQuick) {
      int32_t nx = INT32_MAX;
      for (int e = threadIdx.x; e < TPX; e += NT) {
        const int32_t k = key[e];
        if (k > prev && k < nx) nx = k;  // INT32_MAX (no unit) never qualifies as < nx
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nx = min(nx, __shfl_xor_sync(0xffffffffu, nx, o));
      __syncthreads();  // every thread is done with the previous s_next
      if (threadIdx.x == 0) s_next = INT32_MAX;
      __syncthreads();
      if ((threadIdx.x & 31) == 0) atomicMin(&s_next, nx);
      __syncthreads();
      nx = s_next;
      if (nx == INT32_MAX) break;
      if (total < kQuick && threadIdx.x == 0) s_units[total] = nx;
      ++total;
      prev = nx;
    }
    if (total <= kQuick) {
      __syncthreads();
      if (threadIdx.x == 0) nslots[t] = total;
      if (threadIdx.x < total) tmp[int64_t(t) * TPX + threadIdx.x] = s_units[threadIdx.x];
      for (int e = threadIdx.x; e < TPX; e += NT) {
        const int32_t k = key[e];
        if (k == INT32_MAX) continue;
        int q = 0;
        while (s_units[q] != k) ++q;
        slot[pidx(P, T.y0 + e / TX, T.x0 + e % TX)] = uint16_t(q);
      }
      return;
    }
  }
  __syncthreads();
  for (int k = 2; k <= TPX; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < TPX; i += NT) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int32_t a = key[i], b = key[ixj];
          if ((a > b) == ((i & k) == 0)) {
            key[i] = b;
            key[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  // distinct values: thread owns 8 consecutive sorted entries
  constexpr int PER = TPX / NT;
  int32_t mine[PER];
  int cnt = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = threadIdx.x * PER + q;
    mine[q] = key[e];
    const bool f = mine[q] != INT32_MAX && (e == 0 || mine[q] != key[e - 1]);
    cnt += f;
  }
  int total = 0;
  int pos = block_excl_scan(cnt, sw, total);
  __syncthreads();  // every key read before the distinct list overwrites the front
  // recompute the flags against the previous entry (held by this thread or
  // the previous one) without re-reading the overwritten array
  const int32_t prev_last = __shfl_up_sync(0xffffffffu, mine[PER - 1], 1);
  __shared__ int32_t wlast[NT / 32];
  if ((threadIdx.x & 31) == 31) wlast[threadIdx.x >> 5] = mine[PER - 1];
  __syncthreads();
  int32_t before = (threadIdx.x & 31) ? prev_last
                                      : (threadIdx.x ? wlast[(threadIdx.x >> 5) - 1] : INT32_MIN);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int32_t v = mine[q];
    if (v != INT32_MAX && v != before) {
      key[pos] = v;
      tmp[int64_t(t) * TPX + pos] = v;
      ++pos;
    }
    before = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) nslots[t] = total;
  for (int e = threadIdx.x; e < TPX; e += NT) {
    const int y = T.y0 + e / TX, x = T.x0 + e % TX;
    if (y >= T.y1 || x >= T.x1) continue;
    const int64_t o = pidx(P, y, x);
    const int32_t u = unit[o];
    if (u < 0) continue;
    int lo = 0, hi = total - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (key[mid] < u) lo = mid + 1;
      else hi = mid;
    }
    slot[o] = uint16_t(lo);
  }
}

__global__ void plan_copy_kernel(int ntiles, const int32_t* __restrict__ nslots,
                                 const int32_t* __restrict__ base, const int32_t* __restrict__ tmp,
                                 int32_t* __restrict__ slot_unit, int32_t* __restrict__ tile_flag) {
  const int t = blockIdx.x;
  if (t >= ntiles) return;
  const int n = nslots[t];
  if (threadIdx.x == 0) tile_flag[t] = n > 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    slot_unit[base[t] + k] = tmp[int64_t(t) * TPX + k];
}

__global__ void tile_list_kernel(int ntiles, const int32_t* __restrict__ flag,
                                 const int32_t* __restrict__ pos, int32_t* __restrict__ list) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x)
    if (flag[t]) list[pos[t]] = t;
}

// unit_pstart[u] = first position of unit u in the sorted slot keys
__global__ void unit_bounds_kernel(const int32_t* __restrict__ skeys, int ns, int nu,
                                   int32_t* __restrict__ pstart) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u <= nu; u += gridDim.x * blockDim.x) {
    int lo = 0, hi = ns;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (skeys[mid] < u) lo = mid + 1;
      else hi = mid;
    }
    pstart[u] = lo;
  }
}

__global__ void unit_init_kernel(int nu, const int32_t* __restrict__ unit_comp,
                                 const int32_t* __restrict__ comp_size,
                                 const int32_t* __restrict__ pstart, int cg_max_iters,
                                 uint8_t* __restrict__ status, uint8_t* __restrict__ upd,
                                 int32_t* __restrict__ iters, int32_t* __restrict__ cap,
                                 float* __restrict__ alpha_f, float* __restrict__ beta_f) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += gridDim.x * blockDim.x) {
    const int c = unit_comp ? unit_comp[u] : u;
    const int n = comp_size[c];
    status[u] = pstart[u + 1] > pstart[u] ? U_ACTIVE : U_IDLE;
    upd[u] = 0;
    iters[u] = 0;
    cap[u] = n > cg_max_iters ? n : cg_max_iters;
    alpha_f[u] = 0.f;
    beta_f[u] = 0.f;
  }
}

// ------------------------------------------------------ level construction

constexpr int16_t kNoLink = -32768;
struct alignas(16) Link8 {
  int16_t rel[8];
  __nv_bfloat16 c[8];
};

struct Level {
  int n = 0;        // unknowns
  int nact = 0;     // unknowns with a link (diag > 0)
  int Hb = 0, Wb = 0;  // block grid per map
  int64_t nblk = 0;
  int32_t* bstart = nullptr;  // [nblk + 1]
  int32_t* blk = nullptr;     // [n] block id
  int32_t* unit = nullptr;    // [n]
  int32_t* nbr = nullptr;     // [8][n]
  float* cond = nullptr;      // [8][n]
  float* dinv = nullptr;      // [n]
  int32_t* parent = nullptr;  // [n] (-1: no coarser aggregate)
  int32_t* child = nullptr;   // [4][n] (levels >= 2)
  float* b = nullptr;         // [n]
  float* x1 = nullptr;        // [n] pre-smoothed OM dinv b
  float* x2 = nullptr;        // [n] x1 + OC * parent's correction
  float* e = nullptr;         // [n] (level 1 only)
  Link8* lnk = nullptr;       // [n] compact links (when cmp)
  bool cmp = false;
  int32_t* cnt = nullptr;     // [nblk + 1] scratch (count per block)
};

// distinct values of up to 4 entries (-1 = none), ascending; returns count
__device__ __forceinline__ int distinct4(int32_t v[4], int32_t out[4]) {
  int n = 0;
#pragma unroll
  for (int pass = 0; pass < 4; ++pass) {
    int32_t best = INT32_MAX;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (v[q] >= 0 && v[q] < best && (n == 0 || v[q] > out[n - 1])) best = v[q];
    if (best == INT32_MAX) break;
    out[n++] = best;
  }
  return n;
}

// level 1 from the pixel grid: count units per 2x2 block
__global__ void l1_count_kernel(int B, int H, int W, int P, int Hb, int Wb,
                                const int32_t* __restrict__ unit, int32_t* __restrict__ cnt) {
  const int64_t nblk = int64_t(B) * Hb * Wb;
  for (int64_t bi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; bi < nblk;
       bi += int64_t(gridDim.x) * blockDim.x) {
    const int bx = int(uint32_t(bi) % uint32_t(Wb));
    const int br = int(uint32_t(bi) / uint32_t(Wb));
    const int by = int(br % Hb), m = int(br / Hb);
    int32_t v[4], d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int yy = 2 * by + (q >> 1), xx = 2 * bx + (q & 1);
      v[q] = (yy < H && xx < W) ? unit[pidx(P, m * H + yy, xx)] : -1;
    }
    cnt[bi] = distinct4(v, d);
  }
}

__global__ void l1_assign_kernel(int B, int H, int W, int P, int Hb, int Wb,
                                 const int32_t* __restrict__ unit,
                                 const int32_t* __restrict__ bstart, int32_t* __restrict__ blk,
                                 int32_t* __restrict__ lunit, int32_t* __restrict__ par0) {
  const int64_t nblk = int64_t(B) * Hb * Wb;
  for (int64_t bi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; bi < nblk;
       bi += int64_t(gridDim.x) * blockDim.x) {
    const int bx = int(uint32_t(bi) % uint32_t(Wb));
    const int br = int(uint32_t(bi) / uint32_t(Wb));
    const int by = int(br % Hb), m = int(br / Hb);
    int32_t v[4], d[4];
    int64_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int yy = 2 * by + (q >> 1), xx = 2 * bx + (q & 1);
      const bool in = yy < H && xx < W;
      o[q] = in ? pidx(P, m * H + yy, xx) : -1;
      v[q] = in ? unit[o[q]] : -1;
    }
    const int n = distinct4(v, d);
    const int32_t s0 = bstart[bi];
    for (int k = 0; k < n; ++k) {
      blk[s0 + k] = int32_t(bi);
      lunit[s0 + k] = d[k];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (v[q] < 0) continue;
      int k = 0;
      while (d[k] != v[q]) ++k;
      par0[o[q]] = s0 + k;
    }
  }
}

// unknown of unit u in block bi of a level (-1 if none)
__device__ __forceinline__ int32_t find_in_block(const int32_t* __restrict__ bstart,
                                                 const int32_t* __restrict__ lunit, int64_t bi,
                                                 int32_t u) {
  const int32_t a = bstart[bi], b = bstart[bi + 1];
  for (int32_t k = a; k < b; ++k) {
    const int32_t v = lunit[k];
    if (v == u) return k;
    if (v > u) break;
  }
  return -1;
}

__device__ __forceinline__ void find_neighbours(const int32_t* __restrict__ bstart,
                                                const int32_t* __restrict__ lunit, int32_t bi,
                                                int Hb, int Wb, int32_t u, int32_t* __restrict__ nbr,
                                                int n, int i) {
  const int bx = bi % Wb;
  const int br = bi / Wb;
  const int by = br % Hb;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const int nx = bx + dir_dx(d), ny = by + dir_dy(d);
    int32_t j = -1;
    if (nx >= 0 && nx < Wb && ny >= 0 && ny < Hb)
      j = find_in_block(bstart, lunit, int64_t(bi) + int64_t(dir_dy(d)) * Wb + dir_dx(d), u);
    nbr[int64_t(d) * n + i] = j;
  }
}

// level-1 links: neighbours + Galerkin conductances from the pixel stencil
template <int CONN>
__global__ void l1_links_kernel(int n, int H, int W, int P, int Hb, int Wb,
                                const int32_t* __restrict__ bstart,
                                const int32_t* __restrict__ blk, const int32_t* __restrict__ lunit,
                                const int32_t* __restrict__ unit, const float* __restrict__ hw,
                                const uint8_t* __restrict__ imask, int32_t* __restrict__ nbr,
                                float* __restrict__ cond, float* __restrict__ dinv,
                                int32_t* __restrict__ nact) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  int act = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t bi = blk[i], u = lunit[i];
    find_neighbours(bstart, lunit, bi, Hb, Wb, u, nbr, n, i);
    const int bx = bi % Wb;
    const int br = bi / Wb;
    const int by = br % Hb, m = br / Hb;
    float c[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) c[d] = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int yy = 2 * by + (q >> 1), xx = 2 * bx + (q & 1);
      if (yy >= H || xx >= W) continue;
      const int64_t o = pidx(P, m * H + yy, xx);
      if (unit[o] != u) continue;
      const uint8_t mk = imask[o];
      const float h = hw[o];
#pragma unroll
      for (int bit = 0; bit < 8; ++bit) {
        if ((bit & 3) >= KF || !((mk >> bit) & 1)) continue;
        const int k = bit & 3;
        const int du = bit < 4 ? fwd_du(CONN, k) : -fwd_du(CONN, k);
        const int dv = bit < 4 ? fwd_dv(CONN, k) : -fwd_dv(CONN, k);
        const int jy = yy + dv, jx = xx + du;
        const int dbx = (jx >> 1) - bx, dby = (jy >> 1) - by;  // jx, jy >= 0 (edge inside the map)
        if (dbx == 0 && dby == 0) continue;
        c[dir_of(dbx, dby)] += h + hw[o + int64_t(dv) * P + du];
      }
    }
    float diag = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      cond[int64_t(d) * n + i] = c[d];
      diag += c[d];
    }
    dinv[i] = diag > 0.f ? 1.0f / diag : 0.f;
    act += diag > 0.f;
  }
  act = warp_sum_int(act);
  if ((threadIdx.x & 31) == 0 && act) atomicAdd(nact, act);
}

// level l+1 from level l: count units (with links) over the 2x2 child blocks
__device__ __forceinline__ int merge_children(const int32_t* __restrict__ bstart,
                                              const int32_t* __restrict__ lunit,
                                              const float* __restrict__ dinv, int64_t cb[4],
                                              int32_t* __restrict__ out_units, int out_cap) {
  // 4-way merge of the children blocks' sorted unit lists; only unknowns
  // with a link take part (isolated ones have no coarser aggregate)
  int32_t h[4], e[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    h[q] = cb[q] >= 0 ? bstart[cb[q]] : 0;
    e[q] = cb[q] >= 0 ? bstart[cb[q] + 1] : 0;
  }
  int n = 0;
  while (true) {
    int32_t best = INT32_MAX;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      while (h[q] < e[q] && dinv[h[q]] == 0.f) ++h[q];
      if (h[q] < e[q]) best = min(best, lunit[h[q]]);
    }
    if (best == INT32_MAX) break;
    if (n < out_cap) out_units[n] = best;
    ++n;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (h[q] < e[q] && lunit[h[q]] == best) ++h[q];
  }
  return n;
}

__device__ __forceinline__ void child_blocks(int64_t bi, int Hb, int Wb, int Hc, int Wc,
                                             int64_t cb[4]) {
  const int bx = int(uint32_t(bi) % uint32_t(Wb));
  const int br = int(uint32_t(bi) / uint32_t(Wb));
  const int by = int(br % Hb), m = int(br / Hb);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int cy = 2 * by + (q >> 1), cx = 2 * bx + (q & 1);
    cb[q] = (cy < Hc && cx < Wc) ? (int64_t(m) * Hc + cy) * Wc + cx : -1;
  }
}

__global__ void lc_count_kernel(int64_t nblk, int Hb, int Wb, int Hc, int Wc,
                                const int32_t* __restrict__ cbstart,
                                const int32_t* __restrict__ clunit,
                                const float* __restrict__ cdinv, int32_t* __restrict__ cnt) {
  for (int64_t bi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; bi < nblk;
       bi += int64_t(gridDim.x) * blockDim.x) {
    int64_t cb[4];
    child_blocks(bi, Hb, Wb, Hc, Wc, cb);
    cnt[bi] = merge_children(cbstart, clunit, cdinv, cb, nullptr, 0);
  }
}

__global__ void lc_assign_kernel(int64_t nblk, int Hb, int Wb, int Hc, int Wc,
                                 const int32_t* __restrict__ cbstart,
                                 const int32_t* __restrict__ clunit,
                                 const float* __restrict__ cdinv,
                                 const int32_t* __restrict__ bstart, int n,
                                 int32_t* __restrict__ blk, int32_t* __restrict__ lunit,
                                 int32_t* __restrict__ child, int32_t* __restrict__ cparent) {
  for (int64_t bi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; bi < nblk;
       bi += int64_t(gridDim.x) * blockDim.x) {
    const int32_t s0 = bstart[bi], s1 = bstart[bi + 1];
    if (s0 == s1) continue;
    int64_t cb[4];
    child_blocks(bi, Hb, Wb, Hc, Wc, cb);
    int32_t h[4], e[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = cb[q] >= 0 ? cbstart[cb[q]] : 0;
      e[q] = cb[q] >= 0 ? cbstart[cb[q] + 1] : 0;
    }
    for (int32_t k = s0; k < s1; ++k) {
      int32_t best = INT32_MAX;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        while (h[q] < e[q] && cdinv[h[q]] == 0.f) ++h[q];
        if (h[q] < e[q]) best = min(best, clunit[h[q]]);
      }
      blk[k] = int32_t(bi);
      lunit[k] = best;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int32_t c = -1;
        if (h[q] < e[q] && clunit[h[q]] == best) {
          c = h[q];
          cparent[c] = k;
          ++h[q];
        }
        child[int64_t(q) * n + k] = c;
      }
    }
  }
}

__global__ void lc_links_kernel(int n, int Hb, int Wb, const int32_t* __restrict__ bstart,
                                const int32_t* __restrict__ blk,
                                const int32_t* __restrict__ lunit,
                                const int32_t* __restrict__ child, int nc,
                                const int32_t* __restrict__ cnbr,
                                const float* __restrict__ ccond,
                                const int32_t* __restrict__ cparent, int32_t* __restrict__ nbr,
                                float* __restrict__ cond, float* __restrict__ dinv,
                                int32_t* __restrict__ nact) {
  int act = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t bi = blk[i], u = lunit[i];
    find_neighbours(bstart, lunit, bi, Hb, Wb, u, nbr, n, i);
    const int bx = bi % Wb, by = (bi / Wb) % Hb;
    float c[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) c[d] = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int32_t ch = child[int64_t(q) * n + i];
      if (ch < 0) continue;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int32_t nb = cnbr[int64_t(k) * nc + ch];
        if (nb < 0) continue;
        const float ck = ccond[int64_t(k) * nc + ch];
        if (ck == 0.f) continue;
        const int32_t pj = cparent[nb];
        if (pj < 0 || pj == i) continue;
        const int32_t bj = blk[pj];
        const int dbx = bj % Wb - bx, dby = (bj / Wb) % Hb - by;
        c[dir_of(dbx, dby)] += ck;
      }
    }
    float diag = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      cond[int64_t(d) * n + i] = c[d];
      diag += c[d];
    }
    dinv[i] = diag > 0.f ? 1.0f / diag : 0.f;
    act += diag > 0.f;
  }
  act = warp_sum_int(act);
  if ((threadIdx.x & 31) == 0 && act) atomicAdd(nact, act);
}

// ------------------------------------------------------------ V-cycle

// Compact coarse links: per unknown 32 contiguous bytes, 8 int16 offsets to
// the neighbour (j - i; -32768 = no link) and 8 bf16 conductances (two
// 16-byte loads instead of sixteen 4-byte ones; half the bytes of the
// int32 index + fp32 conductance planes, which the next level's
// construction still reads).  The preconditioner only has to be symmetric
// positive definite, not exact: both directions of a link round the same
// fp32 Galerkin sum.

__global__ void compact_links_kernel(int n, const int32_t* __restrict__ nbr,
                                     const float* __restrict__ cond, Link8* __restrict__ out,
                                     int32_t* __restrict__ overflow) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    Link8 l;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int32_t j = nbr[int64_t(k) * n + i];
      const int32_t d = j - i;
      l.rel[k] = kNoLink;
      l.c[k] = __float2bfloat16_rn(0.f);
      if (j < 0) continue;
      if (d < -32767 || d > 32767) {
        bad = true;
        continue;
      }
      l.rel[k] = int16_t(d);
      l.c[k] = __float2bfloat16_rn(cond[int64_t(k) * n + i]);
    }
    out[i] = l;
    if (bad) atomicOr(overflow, 1);
  }
}

// sum over the links of unknown i: cond * (xi - x[j])
template <bool CMP>
__device__ __forceinline__ float link_sum(int i, int n, const int32_t* __restrict__ nbr,
                                          const float* __restrict__ cond,
                                          const Link8* __restrict__ lnk, float xi,
                                          const float* __restrict__ x) {
  float acc = 0.f;
  if (CMP) {
    const Link8 l = lnk[i];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (l.rel[k] == kNoLink) continue;
      acc += __bfloat162float(l.c[k]) * (xi - x[i + l.rel[k]]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int32_t j = nbr[int64_t(k) * n + i];
      if (j < 0) continue;
      acc += cond[int64_t(k) * n + i] * (xi - x[j]);
    }
  }
  return acc;
}

// down: b_{l+1}[P] = sum over children c of (b - A x1)_c with x1 = OM dinv b
// precomputed at level l; also x1 at level l+1
// Unknowns of units that already converged are skipped (the preconditioner is
// block-diagonal over units, so their stale values never reach a live unit).
template <bool CMP>
__global__ void __launch_bounds__(256) down_kernel(int n1, const int32_t* __restrict__ child,
                                                   int n, const int32_t* __restrict__ nbr,
                                                   const float* __restrict__ cond,
                                                   const Link8* __restrict__ lnk,
                                                   const float* __restrict__ x1,
                                                   const float* __restrict__ b,
                                                   const float* __restrict__ dinv1,
                                                   float* __restrict__ b1,
                                                   float* __restrict__ x1n,
                                                   const int32_t* __restrict__ unit1,
                                                   const uint8_t* __restrict__ status) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += gridDim.x * blockDim.x) {
    if (status[unit1[i]] != U_ACTIVE) continue;
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int32_t c = child[int64_t(q) * n1 + i];
      if (c < 0) continue;
      const float xc = x1[c];
      sum += b[c] - link_sum<CMP>(c, n, nbr, cond, lnk, xc, x1);
    }
    b1[i] = sum;
    x1n[i] = OM * dinv1[i] * sum;
  }
}

// up: e = xs + OM dinv (b - A xs), xs = x2 = x1 + OC e_{l+1}[parent] (x1 on
// the coarsest level); levels >= 2 hand x2 = x1 + OC e to their children.
template <bool SCATTER, bool CMP>
__global__ void __launch_bounds__(256) up_kernel(int n, const int32_t* __restrict__ nbr,
                                                 const float* __restrict__ cond,
                                                 const Link8* __restrict__ lnk,
                                                 const float* __restrict__ dinv,
                                                 const float* __restrict__ b,
                                                 const float* __restrict__ xs,
                                                 float* __restrict__ e_out,
                                                 const int32_t* __restrict__ child,
                                                 const float* __restrict__ x1c,
                                                 float* __restrict__ x2c, int nc,
                                                 const int32_t* __restrict__ unit,
                                                 const uint8_t* __restrict__ status) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (status[unit[i]] != U_ACTIVE) continue;
    const float di = dinv[i];
    float e = 0.f;
    if (di != 0.f) {
      const float xi = xs[i];
      e = xi + OM * di * (b[i] - link_sum<CMP>(i, n, nbr, cond, lnk, xi, xs));
    }
    if (SCATTER) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int32_t c = child[int64_t(q) * n + i];
        if (c >= 0) x2c[c] = x1c[c] + OC * e;
      }
    } else {
      e_out[i] = e;
    }
  }
}

// ---- the small levels in one launch
//
// Below a few thousand unknowns a level's kernels are pure launch latency
// (~3 us each, four per level and V-cycle).  One 1024-thread CTA runs every
// level from the first one with <= kTailMaxN unknowns down to the coarsest and
// back up: the same per-unknown arithmetic as down_kernel / up_kernel (so the
// result does not depend on which levels the tail covers: a batch and its
// single maps stay bit-identical), block barriers instead of launches.
// Unknowns of converged units are not skipped here (their values never reach a
// live unit and stay finite).  The level arrays are written and re-read inside
// the kernel, so nothing here is __restrict__ / read through the non-coherent
// path.
constexpr int kTailThreads = 1024;
#ifndef NI_MG_TAIL_MAX
#define NI_MG_TAIL_MAX 8192
#endif
constexpr int kTailMaxN = NI_MG_TAIL_MAX;
constexpr int kTailMaxLevels = 16;

struct TailLevel {
  int n;
  const Link8* lnk;
  const float* dinv;
  const int32_t* child;  // [4][n]
  float *b, *x1, *x2, *e;
};

struct TailArgs {
  int nlev;            // levels in the tail: lv[1..nlev] = levels T..L
  int nu2;             // 2: two sweeps before / after the coarse correction
  TailLevel lv[kTailMaxLevels + 1];  // lv[0] = level T - 1 (x2 and its pre-smoothed state only)
  const float* xpre0;  // pre-smoothed state of level T - 1
};

__device__ __forceinline__ float tail_link_sum(const TailLevel& V, int i, float xi,
                                               const float* x) {
  float acc = 0.f;
  const Link8 l = V.lnk[i];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (l.rel[k] == kNoLink) continue;
    acc += __bfloat162float(l.c[k]) * (xi - x[i + l.rel[k]]);
  }
  return acc;
}

// xs + OM dinv (b - A xs) at unknown i (up_kernel's expression)
__device__ __forceinline__ float tail_sweep(const TailLevel& V, int i, const float* xs) {
  const float di = V.dinv[i];
  float e = 0.f;
  if (di != 0.f) {
    const float xi = xs[i];
    e = xi + OM * di * (V.b[i] - tail_link_sum(V, i, xi, xs));
  }
  return e;
}

__global__ void __launch_bounds__(kTailThreads) tail_kernel(const __grid_constant__ TailArgs a) {
  const int tid = threadIdx.x;
  for (int k = 1; k <= a.nlev; ++k) {  // down
    const TailLevel& V = a.lv[k];
    const float* xp = V.x1;
    if (a.nu2 == 2) {
      for (int i = tid; i < V.n; i += kTailThreads) V.e[i] = tail_sweep(V, i, V.x1);
      __syncthreads();
      xp = V.e;
    }
    if (k < a.nlev) {
      const TailLevel& N = a.lv[k + 1];
      for (int i = tid; i < N.n; i += kTailThreads) {
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int32_t c = N.child[int64_t(q) * N.n + i];
          if (c < 0) continue;
          const float xc = xp[c];
          sum += V.b[c] - tail_link_sum(V, c, xc, xp);
        }
        N.b[i] = sum;
        N.x1[i] = OM * N.dinv[i] * sum;
      }
      __syncthreads();
    }
  }
  for (int k = a.nlev; k >= 1; --k) {  // up
    const TailLevel& V = a.lv[k];
    const float* xs = k == a.nlev ? (a.nu2 == 2 ? V.e : V.x1) : V.x2;
    if (a.nu2 == 2) {
      for (int i = tid; i < V.n; i += kTailThreads) V.x1[i] = tail_sweep(V, i, xs);
      __syncthreads();
      xs = V.x1;
    }
    const TailLevel& P = a.lv[k - 1];
    const float* xpc = k == 1 ? a.xpre0 : (a.nu2 == 2 ? P.e : P.x1);
    for (int i = tid; i < V.n; i += kTailThreads) {
      const float e = tail_sweep(V, i, xs);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int32_t c = V.child[int64_t(q) * V.n + i];
        if (c >= 0) P.x2[c] = xpc[c] + OC * e;
      }
    }
    __syncthreads();
  }
}

// ---- fine passes
//
// A CTA owns one 64 x 32 tile.  The planes it stencils are staged in shared
// memory as dense boxes (row stride BW, 16-B multiple): by the Tensor Memory
// Accelerator (cp.async.bulk.tensor, one elected thread, an mbarrier with
// the expected byte count; out-of-range rows/columns zero-filled) or, in the
// NI_MG_TMA=0 build, by cp.async (LDGSTS) element copies -- the two variants
// compared in DESIGN.md.  Warp w owns tile rows {2w, 2w+1, 2w+16, 2w+17} and
// lane l the columns l and l+32: consecutive lanes touch consecutive shared
// addresses (no bank conflicts) and every global access is a 128-B row
// segment.  A 2 x 2 block (restriction) is split over lanes l, l^1.
#ifndef NI_MG_TMA
#define NI_MG_TMA 1
#endif
#ifndef NI_MG_V2
#define NI_MG_V2 1  // register-blocked fine passes
#endif
#ifndef NI_MG_CMP_LINKS
#define NI_MG_CMP_LINKS 1  // int16 offsets + bf16 conductances on the coarse levels
#endif
#ifndef NI_MG_B_V2
#define NI_MG_B_V2 0  // register-blocked pass B (measured slower than the scalar pass B)
#endif
#ifndef NI_MG_B2_MINB
#define NI_MG_B2_MINB 2
#endif
#ifndef NI_MG_A2_MINB
#define NI_MG_A2_MINB 3  // resident pass-A CTAs per SM the register budget is cut for
#endif

// TMA boxes must start on a 16-byte-aligned column (measured: an unaligned
// start raises an illegal-instruction fault), so every f32 box starts 4
// columns left of the tile (CX) and every uint8 box 16 columns left (CXM).
constexpr int CX = 4;
constexpr int BW = TX + 2 * CX;  // f32 box width (72: covers a 1- and a 2-pixel halo)
constexpr int BH1 = TY + 2;      // rows with a 1-pixel halo
constexpr int BH2 = TY + 4;      // rows with a 2-pixel halo
constexpr int CXM = 16;
constexpr int BWM = 96;          // uint8 imask box width (x0-16 .. x0+79)
constexpr int S3 = TX + 2;       // x3 array (computed, not a box): 1-pixel halo
constexpr int BOX1 = BW * BH1, BOX2 = BW * BH2;

__host__ __device__ constexpr int al128(int b) { return (b + 127) & ~127; }

struct TmaMaps {
  CUtensorMap r[2], s[2], w, dinv, hw;  // f32, BW x BH1 boxes (pass A)
  CUtensorMap rB[2], dinvB, hwB, parB;  // BW x BH2 boxes (pass B)
  CUtensorMap imB;                      // uint8 imask, BWM x BH1 box (pass B)
  CUtensorMap uI, pI, xI;               // f32, TX x TY interior boxes (pass A v2)
};

struct FineArgs {
  int H, W, P, nTX, nTY;
  int par;  // which r / s buffer holds the values before this iteration's update
  const int32_t* tiles;  // active tiles
  float *x, *p, *u, *w;
  float* rbuf[2];  // r, s ping-pong: neighbouring tiles read the old values as halo
  float* sbuf[2];
  const float *hw, *dinv;
  const uint8_t* imask;
  const int32_t* par0;
  const int32_t* unit;  // padded unit plane (-1 off the units)
  const uint16_t* slot;
  const int32_t* slot_base;  // [ntiles]
  const int32_t* slot_unit;  // [NS]
  const uint8_t* status;
  const uint8_t* upd;
  const float *alpha, *beta;
  float* b1;       // level-1 right-hand side
  float* x1_1;     // level-1 pre-smoothed state OM dinv b
  const float* dinv1;
  const float* e1; // level-1 correction
  double* partial; // [NS][NPART]
  const float* umean;  // per unit: mean of u (removed from p: the preconditioned
                       // direction is kept orthogonal to the unit's null space)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

// cp.async staging of a BWxBH box of a 4-byte plane (NI_MG_TMA=0 variant);
// box rows/columns beyond the padded plane never occur (margins cover them)
template <int BWX, int BHX, class T>
__device__ __forceinline__ void stage_cp(T* sm, const T* g, int P, int ys, int xs) {
  for (int ry = threadIdx.x >> 5; ry < BHX; ry += NT / 32)
    for (int rx = threadIdx.x & 31; rx < BWX; rx += 32)
      cp_async4(sm + ry * BWX + rx, g + pidx(P, ys + ry, xs + rx));
}

// is every unit of the tile finished?  (then its passes are skipped)
__device__ __forceinline__ bool tile_done(const FineArgs& a, int t) {
  const int s0 = a.slot_base[t], s1 = a.slot_base[t + 1];
  for (int k = s0; k < s1; ++k)
    if (a.status[a.slot_unit[k]] == U_ACTIVE) return false;
  return true;
}

// r after the pending update of its unit: r - alpha (w + beta s)
__device__ __forceinline__ float r_new(float r, float w, float s, float al, float bt) {
  return r - al * (w + bt * s);
}

constexpr int kMaxSlotSm = 16;  // per-tile unit scalars kept in shared memory

constexpr size_t kPassASmem = 5 * size_t(al128(BOX1 * 4)) + 128;

// Pass A: pending CG update, pre-smoothing of the new r, residual,
// restriction to level 1.
template <int CONN>
__global__ void __launch_bounds__(NT) pass_a_kernel(const __grid_constant__ FineArgs a,
                                                    const __grid_constant__ TmaMaps tm) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sR = reinterpret_cast<float*>(smem_raw);
  float* sW = sR + al128(BOX1 * 4) / 4;
  float* sS = sW + al128(BOX1 * 4) / 4;
  float* sD = sS + al128(BOX1 * 4) / 4;
  float* sH = sD + al128(BOX1 * 4) / 4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sH + al128(BOX1 * 4) / 4);
  __shared__ float s_al[kMaxSlotSm], s_bt[kMaxSlotSm], s_um[kMaxSlotSm];
  __shared__ int s_un[kMaxSlotSm];
  __shared__ uint8_t s_up[kMaxSlotSm];
  const int t = a.tiles[blockIdx.x];
  if (tile_done(a, t)) return;
  const Tile T = tile_of(t, a.H, a.W, a.nTX, a.nTY);
  const int xs = T.x0 - CX + XM, ys = T.y0 - 1 + RM;  // box origin (padded coordinates)
#if NI_MG_TMA
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, 5u * BOX1 * 4u);
    tma_2d(sR, a.par ? &tm.r[1] : &tm.r[0], bar, xs, ys);
    tma_2d(sW, &tm.w, bar, xs, ys);
    tma_2d(sS, a.par ? &tm.s[1] : &tm.s[0], bar, xs, ys);
    tma_2d(sD, &tm.dinv, bar, xs, ys);
    tma_2d(sH, &tm.hw, bar, xs, ys);
  }
#else
  stage_cp<BW, BH1>(sR, a.rbuf[a.par], a.P, T.y0 - 1, T.x0 - CX);
  stage_cp<BW, BH1>(sW, (const float*)a.w, a.P, T.y0 - 1, T.x0 - CX);
  stage_cp<BW, BH1>(sS, a.sbuf[a.par], a.P, T.y0 - 1, T.x0 - CX);
  stage_cp<BW, BH1>(sD, a.dinv, a.P, T.y0 - 1, T.x0 - CX);
  stage_cp<BW, BH1>(sH, a.hw, a.P, T.y0 - 1, T.x0 - CX);
  asm volatile("cp.async.commit_group;" ::: "memory");
#endif
  const int base = a.slot_base[t];
  const int nsl = a.slot_base[t + 1] - base;
  if (threadIdx.x < nsl && threadIdx.x < kMaxSlotSm) {
    const int un = a.slot_unit[base + threadIdx.x];
    s_un[threadIdx.x] = un;
    s_up[threadIdx.x] = a.upd[un];
    s_al[threadIdx.x] = a.alpha[un];
    s_bt[threadIdx.x] = a.beta[un];
    s_um[threadIdx.x] = a.umean[un];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* rout = a.rbuf[a.par ^ 1];
  float* sout = a.sbuf[a.par ^ 1];
  // per-pixel operands from global (issued before the wait)
  uint16_t slv[2][2][2];
  float uv[2][2][2], pv[2][2][2], xv[2][2][2], d1v[2][2][2];
  int32_t pav[2][2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int ly = 2 * wid + 16 * h + j, lx = lane + 32 * c;
        const int y = T.y0 + ly, x = T.x0 + lx;
        slv[h][j][c] = NOSLOT;
        if (y < T.y1 && x < T.x1) {
          const int64_t o = pidx(a.P, y, x);
          slv[h][j][c] = a.slot[o];
          uv[h][j][c] = a.u[o];
          pv[h][j][c] = a.p[o];
          xv[h][j][c] = a.x[o];
          pav[h][j][c] = a.par0[o];
        }
      }
  // the level-1 diagonal of each pixel's aggregate, gathered while the boxes land
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c)
        d1v[h][j][c] = (slv[h][j][c] != NOSLOT && pav[h][j][c] >= 0)
                           ? __ldg(a.dinv1 + pav[h][j][c]) : 0.f;
#if NI_MG_TMA
  __syncthreads();  // barrier init visible; slot scalars staged
  mbar_wait(bar, 0);
#else
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
#endif
  // Box pass, in place, once per pixel of the tile + its 1-pixel ring: the
  // pending update r' = r - alpha (w + beta s), s' = w + beta s of the
  // pixel's own unit, and the pre-smoothed x1 = OM dinv r' (into sD).  The
  // stencil below then reads x1 and hw only.  A ring pixel's unit is the
  // tile's only unit on a single-slot tile; otherwise it is read from the
  // unit plane (ring pixels of units outside the tile are never stencilled).
  {
    const bool single = nsl == 1;
    const bool up0 = single && s_up[0] != 0;
    const float al0 = single ? s_al[0] : 0.f, bt0 = single ? s_bt[0] : 0.f;
    for (int e = threadIdx.x; e < BH1 * (TX + 2); e += NT) {
      const int ry = e / (TX + 2), rx = e - ry * (TX + 2) + CX - 1;
      const int cb = ry * BW + rx;
      bool up = up0;
      float al = al0, bt = bt0;
      if (!single) {
        const int32_t un = a.unit[pidx(a.P, T.y0 - 1 + ry, T.x0 - CX + rx)];
        up = false;
        if (un >= 0) {
          int k = 0;
          const int nk = nsl < kMaxSlotSm ? nsl : kMaxSlotSm;
          while (k < nk && s_un[k] != un) ++k;
          if (k < nk) {
            up = s_up[k] != 0;
            al = s_al[k];
            bt = s_bt[k];
          } else {
            up = a.upd[un] != 0;
            al = a.alpha[un];
            bt = a.beta[un];
          }
        }
      }
      float r = sR[cb];
      if (up) {
        const float w = sW[cb], sv = sS[cb];
        r = r_new(r, w, sv, al, bt);
        sR[cb] = r;
        sS[cb] = w + bt * sv;
      }
      sD[cb] = OM * sD[cb] * r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float res[2][2];
    int32_t par[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        res[j][c] = 0.f;
        par[j][c] = -1;
        const uint16_t sl = slv[h][j][c];
        if (sl == NOSLOT) continue;
        const int ly = 2 * wid + 16 * h + j, lx = lane + 32 * c;
        const int64_t o = pidx(a.P, T.y0 + ly, T.x0 + lx);
        bool up;
        float al, bt, um;
        if (sl < kMaxSlotSm) {
          up = s_up[sl] != 0;
          al = s_al[sl];
          bt = s_bt[sl];
          um = s_um[sl];
        } else {
          const int un = a.slot_unit[base + sl];
          up = a.upd[un] != 0;
          al = a.alpha[un];
          bt = a.beta[un];
          um = a.umean[un];
        }
        const int cc = (ly + 1) * BW + lx + CX;
        const float ri = sR[cc];
        if (up) {
          const float pi = (uv[h][j][c] - um) + bt * pv[h][j][c];
          a.p[o] = pi;
          a.x[o] = xv[h][j][c] + al * pi;
        }
        rout[o] = ri;
        sout[o] = sS[cc];
        const float x1i = sD[cc];
        const float hi = sH[cc];
        const uint8_t mk = a.imask[o];
        float acc = 0.f;
#pragma unroll
        for (int bit = 0; bit < 8; ++bit) {
          if ((bit & 3) >= KF || !((mk >> bit) & 1)) continue;
          const int jn = cc + nb_off<CONN>(bit, BW);
          acc += (hi + sH[jn]) * (x1i - sD[jn]);
        }
        res[j][c] = ri - acc;
        par[j][c] = pav[h][j][c];
      }
    // restriction: lanes 2k (left column) and 2k+1 (right column) share a
    // 2 x 2 block per column half; the even lane writes each distinct
    // level-1 aggregate once, summing in pixel order (top-left, top-right,
    // bottom-left, bottom-right)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float r01 = __shfl_xor_sync(0xffffffffu, res[0][c], 1);
      const float r11 = __shfl_xor_sync(0xffffffffu, res[1][c], 1);
      const int32_t p01 = __shfl_xor_sync(0xffffffffu, par[0][c], 1);
      const int32_t p11 = __shfl_xor_sync(0xffffffffu, par[1][c], 1);
      const float d01 = __shfl_xor_sync(0xffffffffu, d1v[h][0][c], 1);
      const float d11 = __shfl_xor_sync(0xffffffffu, d1v[h][1][c], 1);
      if (lane & 1) continue;
      const float rq[4] = {res[0][c], r01, res[1][c], r11};
      const int32_t pq[4] = {par[0][c], p01, par[1][c], p11};
      const float dq[4] = {d1v[h][0][c], d01, d1v[h][1][c], d11};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (pq[q] < 0) continue;
        bool first = true;
#pragma unroll
        for (int q2 = 0; q2 < q; ++q2)
          if (pq[q2] == pq[q]) first = false;
        if (!first) continue;
        float sum = 0.f;
#pragma unroll
        for (int q2 = q; q2 < 4; ++q2)
          if (pq[q2] == pq[q]) sum += rq[q2];
        a.b1[pq[q]] = sum;
        a.x1_1[pq[q]] = OM * dq[q] * sum;
      }
    }
  }
}

// Pass B: prolongation + post-smoothing -> u = M r; w = A u; per-slot dots
// (r,u), (w,u), (r,r), sum u, sum r, sum w.
// 54 KB: four CTAs per SM.  The per-slot staging of multi-unit tiles (w values
// and slots of the tile's pixels) reuses the dinv and x2 boxes, which are dead
// once x3 is computed.
constexpr size_t kPassBSmem = 4 * size_t(al128(BOX2 * 4)) + size_t(al128(S3 * BH1 * 4)) +
                              size_t(al128(BWM * BH1)) + 128;
static_assert(TPX * 4 <= BOX2 * 4 && TPX * 2 <= BOX2 * 4, "pass B staging must fit the dead boxes");

template <int CONN>
__global__ void __launch_bounds__(NT) pass_b_kernel(const __grid_constant__ FineArgs a,
                                                    const __grid_constant__ TmaMaps tm) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sR = reinterpret_cast<float*>(smem_raw);
  float* sD = sR + al128(BOX2 * 4) / 4;
  float* sH = sD + al128(BOX2 * 4) / 4;
  float* sX2 = sH + al128(BOX2 * 4) / 4;  // par0 lands here, then x2 replaces it
  float* sX3 = sX2 + al128(BOX2 * 4) / 4;
  uint8_t* sM = reinterpret_cast<uint8_t*>(sX3 + al128(S3 * BH1 * 4) / 4);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sM + al128(BWM * BH1));
  float* sWv = sD;                                  // after the x3 barrier: dinv is dead
  uint16_t* sSl = reinterpret_cast<uint16_t*>(sX2);  // ... and so is x2
  __shared__ double sred[NT / 32][NPART];
  const int t = a.tiles[blockIdx.x];
  if (tile_done(a, t)) return;
  const Tile T = tile_of(t, a.H, a.W, a.nTX, a.nTY);
  const float* rcur = a.rbuf[a.par];
#if NI_MG_TMA
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, 3u * BOX2 * 4u + uint32_t(BWM * BH1));
    const int xs2 = T.x0 - CX + XM, ys2 = T.y0 - 2 + RM;
    tma_2d(sR, a.par ? &tm.rB[1] : &tm.rB[0], bar, xs2, ys2);
    tma_2d(sD, &tm.dinvB, bar, xs2, ys2);
    tma_2d(sH, &tm.hwB, bar, xs2, ys2);
    tma_2d(sM, &tm.imB, bar, T.x0 - CXM + XM, T.y0 - 1 + RM);
  }
#else
  stage_cp<BW, BH2>(sR, rcur, a.P, T.y0 - 2, T.x0 - CX);
  stage_cp<BW, BH2>(sD, a.dinv, a.P, T.y0 - 2, T.x0 - CX);
  stage_cp<BW, BH2>(sH, a.hw, a.P, T.y0 - 2, T.x0 - CX);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int e = threadIdx.x; e < BWM * BH1; e += NT) {
    const int ry = e / BWM, rx = e - ry * BWM;
    sM[e] = a.imask[pidx(a.P, T.y0 - 1 + ry, T.x0 - CXM + rx)];
  }
#endif
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // the level-1 correction OC e1[par0] of the thread's box elements: par0
  // and the e1 gathers are issued while the boxes land (off the critical path)
  constexpr int PER2 = (BOX2 + NT - 1) / NT;
  float ev[PER2];
  {
    int32_t pj[PER2];
#pragma unroll
    for (int q = 0; q < PER2; ++q) {
      const int e = threadIdx.x + q * NT;
      const int ry = e / BW, rx = e - ry * BW;
      pj[q] = e < BOX2 ? a.par0[pidx(a.P, T.y0 - 2 + ry, T.x0 - CX + rx)] : -1;
    }
#pragma unroll
    for (int q = 0; q < PER2; ++q) ev[q] = pj[q] >= 0 ? __ldg(a.e1 + pj[q]) : 0.f;
  }
  // slots of the tile (interior), read while the boxes land
  uint16_t slv[2][2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int ly = 2 * wid + 16 * h + j, lx = lane + 32 * c;
        const int y = T.y0 + ly, x = T.x0 + lx;
        slv[h][j][c] = (y < T.y1 && x < T.x1) ? a.slot[pidx(a.P, y, x)] : NOSLOT;
      }
#if NI_MG_TMA
  __syncthreads();
  mbar_wait(bar, 0);
#else
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
#endif
  // x2 = OM dinv r + OC e1[par0] on the 2-pixel halo box
#pragma unroll
  for (int q = 0; q < PER2; ++q) {
    const int e = threadIdx.x + q * NT;
    if (e < BOX2) sX2[e] = OM * sD[e] * sR[e] + OC * ev[q];
  }
  __syncthreads();
  // post-smoothing on the tile + 1-pixel ring: x3 = x2 + OM dinv (r - A x2).
  // The 66 x 34 ring is walked as a flat list (a row-per-warp mapping spent a
  // third of the stencil's instructions on the two lanes of the 65th / 66th
  // column: the pass is issue-bound)
  for (int e = threadIdx.x; e < S3 * BH1; e += NT) {
    const int ry = e / S3, rx = e - ry * S3;  // pixel (ry - 1, rx - 1) of the tile
    const int c2 = (ry + 1) * BW + rx - 1 + CX;
    const uint8_t mk = sM[ry * BWM + rx - 1 + CXM];
    float v = 0.f;
    if (mk) {
      v = sX2[c2];
      const float hi = sH[c2];
      float acc = 0.f;
#pragma unroll
      for (int bit = 0; bit < 8; ++bit) {
        if ((bit & 3) >= KF || !((mk >> bit) & 1)) continue;
        const int jn = c2 + nb_off<CONN>(bit, BW);
        acc += (hi + sH[jn]) * (v - sX2[jn]);
      }
      v += OM * sD[c2] * (sR[c2] - acc);
    }
    sX3[e] = v;
  }
  __syncthreads();
  // u = x3, w = A u on the tile; per-thread partial dots for the tile's
  // first slot, the other slots' pixels staged for the per-slot pass
  const int nsl = a.slot_base[t + 1] - a.slot_base[t];
  double d[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int ly = 2 * wid + 16 * h + j, lx = lane + 32 * c;
        const uint16_t sl = slv[h][j][c];
        float wv = 0.f;
        if (sl != NOSLOT) {
          const int c1 = (ly + 1) * S3 + lx + 1;
          const int c2 = (ly + 2) * BW + lx + CX;
          const uint8_t mk = sM[(ly + 1) * BWM + lx + CXM];
          const float ui = sX3[c1], hi = sH[c2];
#pragma unroll
          for (int bit = 0; bit < 8; ++bit) {
            if ((bit & 3) >= KF || !((mk >> bit) & 1)) continue;
            wv += (hi + sH[c2 + nb_off<CONN>(bit, BW)]) * (ui - sX3[c1 + nb_off<CONN>(bit, S3)]);
          }
          const int64_t o = pidx(a.P, T.y0 + ly, T.x0 + lx);
          a.u[o] = ui;
          a.w[o] = wv;
          if (sl == 0) {
            const double du = double(ui), dr = double(sR[c2]), dw = double(wv);
            d[0] += dr * du;
            d[1] += dw * du;
            d[2] += dr * dr;
            d[3] += du;
            d[4] += dr;
            d[5] += dw;
          }
        }
        if (nsl > 1) {
          sSl[ly * TX + lx] = sl;
          sWv[ly * TX + lx] = wv;
        }
      }
  // slot 0: fixed-order block reduction
#pragma unroll
  for (int k = 0; k < NPART; ++k) d[k] = warp_sum(d[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NPART; ++k) sred[wid][k] = d[k];
  __syncthreads();
  if (threadIdx.x < NPART) {
    double v = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < NT / 32; ++w8) v += sred[w8][threadIdx.x];
    a.partial[NPART * int64_t(a.slot_base[t]) + threadIdx.x] = v;
  }
  if (nsl <= 1) return;
  // slots 1..: warp w sums slots w+1, w+1+8, ... over the tile lane-strided
  for (int sl = wid + 1; sl < nsl; sl += NT / 32) {
    double q[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int e = lane; e < TPX; e += 32) {
      if (sSl[e] != sl) continue;
      const int ly = e / TX, lx = e - ly * TX;
      const double ui = double(sX3[(ly + 1) * S3 + lx + 1]);
      const double ri = double(sR[(ly + 2) * BW + lx + CX]);
      const double wi = double(sWv[e]);
      q[0] += ri * ui;
      q[1] += wi * ui;
      q[2] += ri * ri;
      q[3] += ui;
      q[4] += ri;
      q[5] += wi;
    }
#pragma unroll
    for (int k = 0; k < NPART; ++k) q[k] = warp_sum(q[k]);
    if (lane == 0) {
      double* pp = a.partial + NPART * int64_t(a.slot_base[t] + sl);
#pragma unroll
      for (int k = 0; k < NPART; ++k) pp[k] = q[k];
    }
  }
}

// ---- register-blocked fine passes (v2)
//
// Thread t of a tile CTA owns the 4 x 2 pixel block at tile columns
// 4 (t & 15) .. +3 and rows 2 (t >> 4) .. +1: two whole 2 x 2 level-1 blocks,
// so the restriction needs no shuffles, and the 4 x 6 window of a plane around
// the block comes out of shared memory as 4 float4 + 8 scalars.  Neighbour
// values then live in registers: every stencil weight and difference is a
// compile-time register index (no per-neighbour shared-memory loads).
// Per-lane global traffic is float4 / 8-byte / 4-byte vectors.

struct Blk {
  int lx0, ly0;  // tile column / row of the block's top-left pixel
};
__device__ __forceinline__ Blk blk_of() {
  Blk b;
  b.lx0 = 4 * (threadIdx.x & 15);
  b.ly0 = 2 * (threadIdx.x >> 4);
  return b;
}

// 4 x 6 window (rows ly0-1..ly0+2, columns lx0-1..lx0+4) of a box whose row 0
// is tile row -ROW0 and whose column CX is tile column 0
template <int ROW0>
__device__ __forceinline__ void load_win(const float* box, const Blk& b, float (&v)[4][6]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float* q = box + (b.ly0 - 1 + r + ROW0) * BW + b.lx0 + CX;
    const float4 m = *reinterpret_cast<const float4*>(q);
    v[r][0] = q[-1];
    v[r][1] = m.x;
    v[r][2] = m.y;
    v[r][3] = m.z;
    v[r][4] = m.w;
    v[r][5] = q[4];
  }
}

// sum over the stencil edges of pixel (i, j) of the block: c_ij * (X_c - X_n),
// c_ij = H_c + H_n; selects (not branches) on the edge bits, so a NaN-free
// product is never needed for absent neighbours
template <int CONN>
__device__ __forceinline__ float stencil_at(const float (&X)[4][6], const float (&Hh)[4][6],
                                            uint32_t mk, int i, int j) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  const float xc = X[i + 1][j + 1], hc = Hh[i + 1][j + 1];
  float acc = 0.f;
#pragma unroll
  for (int bit = 0; bit < 8; ++bit) {
    const int k = bit & 3;
    if (k >= KF) continue;
    const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
    const int r = i + 1 + (bit < 4 ? dv : -dv), c = j + 1 + (bit < 4 ? du : -du);
    const float t = (hc + Hh[r][c]) * (xc - X[r][c]);
    acc += ((mk >> bit) & 1u) ? t : 0.f;
  }
  return acc;
}

struct UnitScalars {
  bool up;
  float al, bt, um;
};

constexpr int IBOX = TX * TY;  // interior box (no halo)
constexpr size_t kPassA2Smem = 5 * size_t(al128(BOX1 * 4)) + 3 * size_t(IBOX * 4) + 128;

// Pass A (v2): pending CG update, pre-smoothing of the new r, residual,
// restriction to level 1.  TMA brings the five halo boxes (r, w, s, dinv,
// hw) and the three interior boxes (u, p, x).
// stage buffers of pass A (halo boxes r, w, s, dinv, hw; interior u, p, x)
struct AStage {
  float *sR, *sW, *sS, *sD, *sH, *sU, *sP, *sX;
};
__device__ __forceinline__ AStage astage(unsigned char* base) {
  AStage g;
  g.sR = reinterpret_cast<float*>(base);
  g.sW = g.sR + al128(BOX1 * 4) / 4;
  g.sS = g.sW + al128(BOX1 * 4) / 4;
  g.sD = g.sS + al128(BOX1 * 4) / 4;
  g.sH = g.sD + al128(BOX1 * 4) / 4;
  g.sU = g.sH + al128(BOX1 * 4) / 4;
  g.sP = g.sU + IBOX;
  g.sX = g.sP + IBOX;
  return g;
}
constexpr size_t kAStageBytes = 5 * size_t(al128(BOX1 * 4)) + 3 * size_t(IBOX * 4);

// TMA copies of tile t's pass-A planes into a stage (one elected thread)
__device__ __forceinline__ void a2_issue(const FineArgs& a, const TmaMaps& tm, int t,
                                         const AStage& g, uint64_t* bar) {
  const Tile T = tile_of(t, a.H, a.W, a.nTX, a.nTY);
  const int xs = T.x0 - CX + XM, ys = T.y0 - 1 + RM;  // halo box origin (padded)
  mbar_expect_tx(bar, 5u * BOX1 * 4u + 3u * IBOX * 4u);
  tma_2d(g.sR, a.par ? &tm.r[1] : &tm.r[0], bar, xs, ys);
  tma_2d(g.sW, &tm.w, bar, xs, ys);
  tma_2d(g.sS, a.par ? &tm.s[1] : &tm.s[0], bar, xs, ys);
  tma_2d(g.sD, &tm.dinv, bar, xs, ys);
  tma_2d(g.sH, &tm.hw, bar, xs, ys);
  tma_2d(g.sU, &tm.uI, bar, T.x0 + XM, T.y0 + RM);
  tma_2d(g.sP, &tm.pI, bar, T.x0 + XM, T.y0 + RM);
  tma_2d(g.sX, &tm.xI, bar, T.x0 + XM, T.y0 + RM);
}

struct ASlots {
  float al[kMaxSlotSm], bt[kMaxSlotSm], um[kMaxSlotSm];
  int un[kMaxSlotSm];
  uint8_t up[kMaxSlotSm];
};

// Pass A on tile t whose planes land in stage g (mbarrier bar, parity
// phase): everything after the TMA issue.
template <int CONN>
__device__ __forceinline__ void a2_tile(const FineArgs& a, int t, const AStage& g, uint64_t* bar,
                                        uint32_t phase, ASlots& sc) {
  float* sR = g.sR;
  float* sS = g.sS;
  float* sW = g.sW;
  float* sD = g.sD;
  float* sH = g.sH;
  float* sU = g.sU;
  float* sP = g.sP;
  float* sXv = g.sX;
  float* s_al = sc.al;
  float* s_bt = sc.bt;
  float* s_um = sc.um;
  int* s_un = sc.un;
  uint8_t* s_up = sc.up;
  const Tile T = tile_of(t, a.H, a.W, a.nTX, a.nTY);
  const int base = a.slot_base[t];
  const int nsl = a.slot_base[t + 1] - base;
  if (threadIdx.x < nsl && threadIdx.x < kMaxSlotSm) {
    const int un = a.slot_unit[base + threadIdx.x];
    s_un[threadIdx.x] = un;
    s_up[threadIdx.x] = a.upd[un];
    s_al[threadIdx.x] = a.alpha[un];
    s_bt[threadIdx.x] = a.beta[un];
    s_um[threadIdx.x] = a.umean[un];
  }
  const Blk b = blk_of();
  // the block's slots, level-1 parents and edge masks (issued before the wait)
  bool rowv[2];
  uint16_t sl[2][4];
  int32_t pa[2][4];
  uint32_t mk[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int y = T.y0 + b.ly0 + i;
    rowv[i] = y < T.y1;
    const int64_t o = pidx(a.P, y, T.x0 + b.lx0);
    const ushort4 s4 = *reinterpret_cast<const ushort4*>(a.slot + o);
    const int4 p4 = *reinterpret_cast<const int4*>(a.par0 + o);
    mk[i] = *reinterpret_cast<const uint32_t*>(a.imask + o);
    sl[i][0] = s4.x;
    sl[i][1] = s4.y;
    sl[i][2] = s4.z;
    sl[i][3] = s4.w;
    pa[i][0] = p4.x;
    pa[i][1] = p4.y;
    pa[i][2] = p4.z;
    pa[i][3] = p4.w;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (!rowv[i] || T.x0 + b.lx0 + j >= T.x1) sl[i][j] = NOSLOT;
  }
  __syncthreads();  // barrier init visible; slot scalars staged
  mbar_wait(bar, phase);
  // box pass, in place, float4-wide over the tile + 1-pixel ring (see pass A)
  {
    const bool single = nsl == 1;
    const bool up0 = single && s_up[0] != 0;
    const float al0 = single ? s_al[0] : 0.f, bt0 = single ? s_bt[0] : 0.f;
    constexpr int Q = BW / 4;
    for (int it = threadIdx.x; it < BH1 * Q; it += NT) {
      const int ry = it / Q, q = it - ry * Q;
      const int cb = ry * BW + 4 * q;
      float4 r4 = *reinterpret_cast<float4*>(sR + cb);
      bool up[4] = {up0, up0, up0, up0};
      float al[4] = {al0, al0, al0, al0}, bt[4] = {bt0, bt0, bt0, bt0};
      if (!single) {
        const int4 u4 = *reinterpret_cast<const int4*>(
            a.unit + pidx(a.P, T.y0 - 1 + ry, T.x0 - CX + 4 * q));
        const int32_t uu[4] = {u4.x, u4.y, u4.z, u4.w};
        const int nk = nsl < kMaxSlotSm ? nsl : kMaxSlotSm;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          up[e] = false;
          if (uu[e] < 0) continue;
          int k = 0;
          while (k < nk && s_un[k] != uu[e]) ++k;
          if (k < nk) {
            up[e] = s_up[k] != 0;
            al[e] = s_al[k];
            bt[e] = s_bt[k];
          } else {
            up[e] = a.upd[uu[e]] != 0;
            al[e] = a.alpha[uu[e]];
            bt[e] = a.beta[uu[e]];
          }
        }
      }
      if (up[0] | up[1] | up[2] | up[3]) {
        const float4 w4 = *reinterpret_cast<const float4*>(sW + cb);
        float4 s4 = *reinterpret_cast<float4*>(sS + cb);
        float* rr = &r4.x;
        float* ss = &s4.x;
        const float* ww = &w4.x;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (up[e]) {
            rr[e] = r_new(rr[e], ww[e], ss[e], al[e], bt[e]);
            ss[e] = ww[e] + bt[e] * ss[e];
          }
        *reinterpret_cast<float4*>(sR + cb) = r4;
        *reinterpret_cast<float4*>(sS + cb) = s4;
      }
      float4 d4 = *reinterpret_cast<float4*>(sD + cb);
      d4.x = OM * d4.x * r4.x;
      d4.y = OM * d4.y * r4.y;
      d4.z = OM * d4.z * r4.z;
      d4.w = OM * d4.w * r4.w;
      *reinterpret_cast<float4*>(sD + cb) = d4;
    }
  }
  __syncthreads();
  float* rout = a.rbuf[a.par ^ 1];
  float* sout = a.sbuf[a.par ^ 1];
  float res[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    // window rows i .. i + 2 of the 4 x 6 window (the stencil of output row i)
    float X[4][6], Hh[4][6];
#pragma unroll
    for (int r = i; r < i + 3; ++r) {
      const float* qx = sD + (b.ly0 + r) * BW + b.lx0 + CX;
      const float* qh = sH + (b.ly0 + r) * BW + b.lx0 + CX;
      const float4 mx = *reinterpret_cast<const float4*>(qx);
      const float4 mh = *reinterpret_cast<const float4*>(qh);
      X[r][0] = qx[-1];
      X[r][1] = mx.x;
      X[r][2] = mx.y;
      X[r][3] = mx.z;
      X[r][4] = mx.w;
      X[r][5] = qx[4];
      Hh[r][0] = qh[-1];
      Hh[r][1] = mh.x;
      Hh[r][2] = mh.y;
      Hh[r][3] = mh.z;
      Hh[r][4] = mh.w;
      Hh[r][5] = qh[4];
    }
    const int cb = (b.ly0 + i + 1) * BW + b.lx0 + CX;
    const int ci = (b.ly0 + i) * TX + b.lx0;
    const float4 r4 = *reinterpret_cast<const float4*>(sR + cb);
    const float4 s4 = *reinterpret_cast<const float4*>(sS + cb);
    const float4 u4 = *reinterpret_cast<const float4*>(sU + ci);
    float4 p4 = *reinterpret_cast<const float4*>(sP + ci);
    float4 x4 = *reinterpret_cast<const float4*>(sXv + ci);
    const float* rr = &r4.x;
    const float* uu = &u4.x;
    float* pp = &p4.x;
    float* xx = &x4.x;
    bool any = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      res[i][j] = 0.f;
      const uint16_t q = sl[i][j];
      if (q == NOSLOT) continue;
      UnitScalars us;
      if (nsl == 1) {  // most tiles: one unit, its scalars hoisted by the compiler
        us.up = s_up[0] != 0;
        us.al = s_al[0];
        us.bt = s_bt[0];
        us.um = s_um[0];
      } else if (q < kMaxSlotSm) {
        us.up = s_up[q] != 0;
        us.al = s_al[q];
        us.bt = s_bt[q];
        us.um = s_um[q];
      } else {
        const int un = a.slot_unit[base + q];
        us.up = a.upd[un] != 0;
        us.al = a.alpha[un];
        us.bt = a.beta[un];
        us.um = a.umean[un];
      }
      if (us.up) {
        pp[j] = (uu[j] - us.um) + us.bt * pp[j];
        xx[j] = xx[j] + us.al * pp[j];
        any = true;
      }
      res[i][j] = rr[j] - stencil_at<CONN>(X, Hh, (mk[i] >> (8 * j)) & 0xffu, i, j);
    }
    if (rowv[i]) {
      const int64_t o = pidx(a.P, T.y0 + b.ly0 + i, T.x0 + b.lx0);
      *reinterpret_cast<float4*>(rout + o) = r4;
      *reinterpret_cast<float4*>(sout + o) = s4;
      if (any) {
        *reinterpret_cast<float4*>(a.p + o) = p4;
        *reinterpret_cast<float4*>(a.x + o) = x4;
      }
    }
  }
  // restriction: the two 2 x 2 blocks of the thread, each distinct level-1
  // aggregate written once, summed in pixel order (TL, TR, BL, BR)
#pragma unroll
  for (int hb = 0; hb < 2; ++hb) {
    const float rq[4] = {res[0][2 * hb], res[0][2 * hb + 1], res[1][2 * hb], res[1][2 * hb + 1]};
    int32_t pq[4] = {pa[0][2 * hb], pa[0][2 * hb + 1], pa[1][2 * hb], pa[1][2 * hb + 1]};
    const uint16_t sq[4] = {sl[0][2 * hb], sl[0][2 * hb + 1], sl[1][2 * hb], sl[1][2 * hb + 1]};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (sq[q] == NOSLOT) pq[q] = -1;
    if (pq[0] >= 0 && pq[1] == pq[0] && pq[2] == pq[0] && pq[3] == pq[0]) {
      // the common case: one aggregate for the whole block (same order as below)
      const float sum = ((rq[0] + rq[1]) + rq[2]) + rq[3];
      a.b1[pq[0]] = sum;
      a.x1_1[pq[0]] = OM * __ldg(a.dinv1 + pq[0]) * sum;
      continue;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (pq[q] < 0) continue;
      bool first = true;
#pragma unroll
      for (int q2 = 0; q2 < q; ++q2)
        if (pq[q2] == pq[q]) first = false;
      if (!first) continue;
      float sum = 0.f;
#pragma unroll
      for (int q2 = q; q2 < 4; ++q2)
        if (pq[q2] == pq[q]) sum += rq[q2];
      a.b1[pq[q]] = sum;
      a.x1_1[pq[q]] = OM * __ldg(a.dinv1 + pq[q]) * sum;
    }
  }
}

// Pass A (v2): pending CG update, pre-smoothing of the new r, residual,
// restriction to level 1; one tile per CTA, TMA brings the five halo boxes
// (r, w, s, dinv, hw) and the three interior boxes (u, p, x).
template <int CONN>
__global__ void __launch_bounds__(NT, NI_MG_A2_MINB) pass_a2_kernel(
    const __grid_constant__ FineArgs a, const __grid_constant__ TmaMaps tm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const AStage g = astage(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + kAStageBytes);
  __shared__ ASlots sc;
  const int t = a.tiles[blockIdx.x];
  if (tile_done(a, t)) return;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    a2_issue(a, tm, t, g, bar);
  }
  a2_tile<CONN>(a, t, g, bar, 0, sc);
}

constexpr size_t kPassB2Smem = 4 * size_t(al128(BOX2 * 4)) + size_t(al128(BOX1 * 4)) +
                               size_t(al128(BWM * BH1)) + size_t(TPX) * 4 + size_t(TPX) * 2 + 128;

// 3 x 6 rows (i .. i + 2) of the 4 x 6 window of a box whose row 0 is tile row
// -ROW0 (see load_win)
template <int ROW0>
__device__ __forceinline__ void load_rows3(const float* box, const Blk& b, int i,
                                           float (&v)[4][6]) {
#pragma unroll
  for (int r = i; r < i + 3; ++r) {
    const float* q = box + (b.ly0 - 1 + r + ROW0) * BW + b.lx0 + CX;
    const float4 m = *reinterpret_cast<const float4*>(q);
    v[r][0] = q[-1];
    v[r][1] = m.x;
    v[r][2] = m.y;
    v[r][3] = m.z;
    v[r][4] = m.w;
    v[r][5] = q[4];
  }
}

// Pass B (v2): prolongation + post-smoothing -> u = M r; w = A u; per-slot dots
// (r,u), (w,u), (r,r), sum u, sum r, sum w.  Same staging as pass B; the
// post-smoothing and A u of the tile interior are register-blocked, the
// 1-pixel ring of x3 is one pixel per thread.
template <int CONN>
__global__ void __launch_bounds__(NT, NI_MG_B2_MINB) pass_b2_kernel(const __grid_constant__ FineArgs a,
                                                       const __grid_constant__ TmaMaps tm) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sR = reinterpret_cast<float*>(smem_raw);
  float* sD = sR + al128(BOX2 * 4) / 4;
  float* sH = sD + al128(BOX2 * 4) / 4;
  float* sX2 = sH + al128(BOX2 * 4) / 4;  // par0 lands here, then x2 replaces it
  float* sX3 = sX2 + al128(BOX2 * 4) / 4;  // BW x BH1: row 0 = tile row -1
  uint8_t* sM = reinterpret_cast<uint8_t*>(sX3 + al128(BOX1 * 4) / 4);
  float* sWv = reinterpret_cast<float*>(sM + al128(BWM * BH1));
  uint16_t* sSl = reinterpret_cast<uint16_t*>(sWv + TPX);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sSl + TPX);
  __shared__ double sred[NT / 32][NPART];
  const int t = a.tiles[blockIdx.x];
  if (tile_done(a, t)) return;
  const Tile T = tile_of(t, a.H, a.W, a.nTX, a.nTY);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, 3u * BOX2 * 4u + uint32_t(BWM * BH1));
    const int xs2 = T.x0 - CX + XM, ys2 = T.y0 - 2 + RM;
    tma_2d(sR, a.par ? &tm.rB[1] : &tm.rB[0], bar, xs2, ys2);
    tma_2d(sD, &tm.dinvB, bar, xs2, ys2);
    tma_2d(sH, &tm.hwB, bar, xs2, ys2);
    tma_2d(sM, &tm.imB, bar, T.x0 - CXM + XM, T.y0 - 1 + RM);
  }
  // OC e1[par0] of the thread's float4 items of the 2-pixel halo box,
  // gathered while the boxes land
  constexpr int QB = BW / 4, NIT = (BH2 * QB + NT - 1) / NT;
  float4 ev[NIT];
#pragma unroll
  for (int q = 0; q < NIT; ++q) {
    const int it = threadIdx.x + q * NT;
    int4 p4 = make_int4(-1, -1, -1, -1);
    if (it < BH2 * QB) {
      const int ry = it / QB, qq = it - ry * QB;
      p4 = *reinterpret_cast<const int4*>(a.par0 + pidx(a.P, T.y0 - 2 + ry, T.x0 - CX + 4 * qq));
    }
    ev[q].x = p4.x >= 0 ? __ldg(a.e1 + p4.x) : 0.f;
    ev[q].y = p4.y >= 0 ? __ldg(a.e1 + p4.y) : 0.f;
    ev[q].z = p4.z >= 0 ? __ldg(a.e1 + p4.z) : 0.f;
    ev[q].w = p4.w >= 0 ? __ldg(a.e1 + p4.w) : 0.f;
  }
  const Blk b = blk_of();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool rowv[2];
  uint16_t sl[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int y = T.y0 + b.ly0 + i;
    rowv[i] = y < T.y1;
    const ushort4 s4 = *reinterpret_cast<const ushort4*>(a.slot + pidx(a.P, y, T.x0 + b.lx0));
    sl[i][0] = s4.x;
    sl[i][1] = s4.y;
    sl[i][2] = s4.z;
    sl[i][3] = s4.w;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (!rowv[i] || T.x0 + b.lx0 + j >= T.x1) sl[i][j] = NOSLOT;
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // x2 = OM dinv r + OC e1[par0] on the 2-pixel halo box, float4-wide
#pragma unroll
  for (int q = 0; q < NIT; ++q) {
    const int it = threadIdx.x + q * NT;
    if (it >= BH2 * QB) continue;
    const int cb = it * 4;  // rows are BW = 4 QB floats: item it covers [4 it, 4 it + 4)
    const float4 r4 = *reinterpret_cast<const float4*>(sR + cb);
    const float4 d4 = *reinterpret_cast<const float4*>(sD + cb);
    float4 x4;
    x4.x = OM * d4.x * r4.x + OC * ev[q].x;
    x4.y = OM * d4.y * r4.y + OC * ev[q].y;
    x4.z = OM * d4.z * r4.z + OC * ev[q].z;
    x4.w = OM * d4.w * r4.w + OC * ev[q].w;
    *reinterpret_cast<float4*>(sX2 + cb) = x4;
  }
  __syncthreads();
  // post-smoothing x3 = x2 + OM dinv (r - A x2): the 1-pixel ring, one pixel
  // per thread (66 + 66 + 32 + 32 = 196 pixels)
  if (threadIdx.x < 196) {
    int ly, lx;
    const int q = threadIdx.x;
    if (q < 66) {
      ly = -1;
      lx = q - 1;
    } else if (q < 132) {
      ly = TY;
      lx = q - 67;
    } else if (q < 164) {
      ly = q - 132;
      lx = -1;
    } else {
      ly = q - 164;
      lx = TX;
    }
    const int c2 = (ly + 2) * BW + lx + CX;
    const uint8_t mk = sM[(ly + 1) * BWM + lx + CXM];
    float v = 0.f;
    if (mk) {
      v = sX2[c2];
      const float hi = sH[c2];
      float acc = 0.f;
#pragma unroll
      for (int bit = 0; bit < 8; ++bit) {
        if ((bit & 3) >= KF || !((mk >> bit) & 1)) continue;
        const int jn = c2 + nb_off<CONN>(bit, BW);
        acc += (hi + sH[jn]) * (v - sX2[jn]);
      }
      v += OM * sD[c2] * (sR[c2] - acc);
    }
    sX3[(ly + 1) * BW + lx + CX] = v;
  }
  // ... and the interior, register-blocked
  uint32_t mk[2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
    mk[i] = *reinterpret_cast<const uint32_t*>(sM + (b.ly0 + i + 1) * BWM + b.lx0 + CXM);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float X[4][6], Hh[4][6];
    load_rows3<2>(sX2, b, i, X);
    load_rows3<2>(sH, b, i, Hh);
    const int c2 = (b.ly0 + i + 2) * BW + b.lx0 + CX;
    const float4 r4 = *reinterpret_cast<const float4*>(sR + c2);
    const float4 d4 = *reinterpret_cast<const float4*>(sD + c2);
    const float* rr = &r4.x;
    const float* dd = &d4.x;
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t m = (mk[i] >> (8 * j)) & 0xffu;
      const float acc = stencil_at<CONN>(X, Hh, m, i, j);
      const float v = X[i + 1][j + 1] + OM * dd[j] * (rr[j] - acc);
      o[j] = m ? v : 0.f;
    }
    *reinterpret_cast<float4*>(sX3 + (b.ly0 + i + 1) * BW + b.lx0 + CX) =
        make_float4(o[0], o[1], o[2], o[3]);
  }
  __syncthreads();
  // u = x3, w = A u on the interior; per-thread partial dots of slot 0
  const int nsl = a.slot_base[t + 1] - a.slot_base[t];
  double d[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float X[4][6], Hh[4][6];
    load_rows3<1>(sX3, b, i, X);
    load_rows3<2>(sH, b, i, Hh);
    const float4 r4 = *reinterpret_cast<const float4*>(sR + (b.ly0 + i + 2) * BW + b.lx0 + CX);
    const float* rr = &r4.x;
    float wv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t m = (mk[i] >> (8 * j)) & 0xffu;
      wv[j] = stencil_at<CONN>(X, Hh, m, i, j);
      if (sl[i][j] == 0) {
        const double du = double(X[i + 1][j + 1]), dr = double(rr[j]), dw = double(wv[j]);
        d[0] += dr * du;
        d[1] += dw * du;
        d[2] += dr * dr;
        d[3] += du;
        d[4] += dr;
        d[5] += dw;
      }
      if (nsl > 1) {
        sSl[(b.ly0 + i) * TX + b.lx0 + j] = sl[i][j];
        sWv[(b.ly0 + i) * TX + b.lx0 + j] = wv[j];
      }
    }
    if (rowv[i]) {
      const int64_t o = pidx(a.P, T.y0 + b.ly0 + i, T.x0 + b.lx0);
      *reinterpret_cast<float4*>(a.u + o) =
          make_float4(X[i + 1][1], X[i + 1][2], X[i + 1][3], X[i + 1][4]);
      *reinterpret_cast<float4*>(a.w + o) = make_float4(wv[0], wv[1], wv[2], wv[3]);
    }
  }
  // slot 0: fixed-order block reduction
#pragma unroll
  for (int k = 0; k < NPART; ++k) d[k] = warp_sum(d[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NPART; ++k) sred[wid][k] = d[k];
  __syncthreads();
  if (threadIdx.x < NPART) {
    double v = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < NT / 32; ++w8) v += sred[w8][threadIdx.x];
    a.partial[NPART * int64_t(a.slot_base[t]) + threadIdx.x] = v;
  }
  if (nsl <= 1) return;
  // slots 1..: warp w sums slots w+1, w+1+8, ... over the tile lane-strided
  for (int q = wid + 1; q < nsl; q += NT / 32) {
    double qd[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int e = lane; e < TPX; e += 32) {
      if (sSl[e] != q) continue;
      const int ly = e / TX, lx = e - ly * TX;
      const double ui = double(sX3[(ly + 1) * BW + lx + CX]);
      const double ri = double(sR[(ly + 2) * BW + lx + CX]);
      const double wi = double(sWv[e]);
      qd[0] += ri * ui;
      qd[1] += wi * ui;
      qd[2] += ri * ri;
      qd[3] += ui;
      qd[4] += ri;
      qd[5] += wi;
    }
#pragma unroll
    for (int k = 0; k < NPART; ++k) qd[k] = warp_sum(qd[k]);
    if (lane == 0) {
      double* pp = a.partial + NPART * int64_t(a.slot_base[t] + q);
#pragma unroll
      for (int k = 0; k < NPART; ++k) pp[k] = qd[k];
    }
  }
}

// ---- per-unit scalars (warp per unit): scipy's stop test on the recursive
// residual, then the Chronopoulos-Gear alpha / beta
struct ScalarArgs {
  int nu;
  const int32_t* pstart;
  const int32_t* plist;
  const double* partial;
  const double* unit_n;  // pixels per unit
  double rtol;
  uint8_t* status;
  uint8_t* upd;
  int32_t* iters;
  const int32_t* cap;
  double* tol2;
  double* gprev;
  double* aprev;
  float* alpha;
  float* beta;
  float* umean;
  int32_t* nactive;
  unsigned long long* px_done;  // pixels of the units this V-cycle processed
  int trace_unit;  // debug: print this unit's scalars every iteration (-1: off)
};

// The unit's Laplacian is singular (constants); float32 roundoff leaves
// O(eps) null-space components in r and, amplified by the smoother, in
// u = M r.  They carry no information (CG from 0 lives in range(A)) but
// would stall / destabilise the recursion once ||r|| nears 1e-6 ||b||, so
// the preconditioned vector is projected on range(A): u' = u - mean(u)
// (w = A u' = A u in difference form), and the stop test uses the range
// part of r -- the residual float64 arithmetic (the reference) would have.
__global__ void __launch_bounds__(256) scalar_kernel(const __grid_constant__ ScalarArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  int act = 0;
  unsigned long long pxd = 0;
  for (int u = gw; u < a.nu; u += nw) {
    if (a.status[u] != U_ACTIVE) continue;  // warp-uniform
    pxd += (unsigned long long)a.unit_n[u];
    double d[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = a.pstart[u] + lane; k < a.pstart[u + 1]; k += 32) {
      const double* pp = a.partial + NPART * int64_t(a.plist[k]);
#pragma unroll
      for (int q = 0; q < NPART; ++q) d[q] += pp[q];
    }
#pragma unroll
    for (int q = 0; q < NPART; ++q) d[q] = warp_sum(d[q]);
    if (lane == 0) {
      const double n = a.unit_n[u];
      const double cu = d[3] / n;
      const double g = d[0] - cu * d[4];
      const double dl = d[1] - cu * d[5];
      const double rr = fmax(d[2] - d[4] * d[4] / n, 0.0);
      const int it = a.iters[u];
      if (u == a.trace_unit)
        printf("mg unit %d it %d (r,u')=%.6e (w,u')=%.6e |r|=%.6e |r_range|=%.6e mean u=%.3e\n",
               u, it, g, dl, sqrt(d[2]), sqrt(rr), cu);
      if (it == 0) a.tol2[u] = rr;  // ||b||^2 (r = b before the first update)
      const double tol = a.rtol * sqrt(a.tol2[u]);
      uint8_t st = U_ACTIVE, up = 0;
      if (it >= a.cap[u]) {  // scipy: no test after the last allowed update
        st = U_CAPPED;
      } else if (rr == 0.0 || sqrt(rr) < tol) {
        st = U_CONV;
      } else {
        double al, bt;
        if (it == 0) {
          bt = 0.0;
          al = g / dl;
        } else {
          bt = g / a.gprev[u];
          al = g / (dl - bt * g / a.aprev[u]);
        }
        if (!(al > 0.0) || !isfinite(al) || !isfinite(bt)) {
          st = U_CAPPED;  // breakdown (never seen): report like a cap
        } else {
          a.gprev[u] = g;
          a.aprev[u] = al;
          a.alpha[u] = float(al);
          a.beta[u] = float(bt);
          a.umean[u] = float(cu);
          a.iters[u] = it + 1;
          up = 1;
          ++act;
        }
      }
      a.status[u] = st;
      a.upd[u] = up;
    }
  }
  act = warp_sum_int(act);
  if (lane == 0 && act) atomicAdd(a.nactive, act);
  if (lane == 0 && pxd) atomicAdd(a.px_done, pxd);  // lanes of a warp agree on pxd
}

// ---- output: x minus its per-unit mean (the gauge of CG from x0 = 0)
__global__ void __launch_bounds__(NT) xsum_kernel(const __grid_constant__ FineArgs a) {
  __shared__ uint16_t sSl[TPX];
  __shared__ float sX[TPX];
  const int t = a.tiles[blockIdx.x];
  const Tile T = tile_of(t, a.H, a.W, a.nTX, a.nTY);
  for (int e = threadIdx.x; e < TPX; e += NT) {
    const int y = T.y0 + e / TX, x = T.x0 + e % TX;
    uint16_t sl = NOSLOT;
    float xv = 0.f;
    if (y < T.y1 && x < T.x1) {
      const int64_t o = pidx(a.P, y, x);
      sl = a.slot[o];
      xv = a.x[o];
    }
    sSl[e] = sl;
    sX[e] = xv;
  }
  __syncthreads();
  const int nsl = a.slot_base[t + 1] - a.slot_base[t];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int sl = wid; sl < nsl; sl += NT / 32) {
    double sx = 0.0, sn = 0.0;
    for (int e = lane; e < TPX; e += 32) {
      if (sSl[e] != sl) continue;
      sx += double(sX[e]);
      sn += 1.0;
    }
    sx = warp_sum(sx);
    sn = warp_sum(sn);
    if (lane == 0) {
      double* pp = a.partial + NPART * int64_t(a.slot_base[t] + sl);
      pp[0] = sx;
      pp[1] = sn;
    }
  }
}

// per unit: mean of x (pp[0] / pp[1]) and, if n_out, its pixel count
__global__ void unit_mean_kernel(int nu, const int32_t* __restrict__ pstart,
                                 const int32_t* __restrict__ plist,
                                 const double* __restrict__ partial, double* __restrict__ mean,
                                 double* __restrict__ n_out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int u = gw; u < nu; u += nw) {
    double sx = 0.0, sn = 0.0;
    for (int k = pstart[u] + lane; k < pstart[u + 1]; k += 32) {
      const double* pp = partial + NPART * int64_t(plist[k]);
      sx += pp[0];
      sn += pp[1];
    }
    sx = warp_sum(sx);
    sn = warp_sum(sn);
    if (lane == 0) {
      mean[u] = sn > 0.0 ? sx / sn : 0.0;
      if (n_out) n_out[u] = sn;
    }
  }
}

__global__ void output_kernel(int W, int P, int64_t npix, const float* __restrict__ x,
                              const int32_t* __restrict__ unit, const double* __restrict__ mean,
                              double* __restrict__ z) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = pidx(P, int(uint32_t(i) / uint32_t(W)), int(uint32_t(i) % uint32_t(W)));
    const int32_t u = unit[o];
    z[i] = u >= 0 ? double(x[o]) - mean[u] : 0.0;
  }
}

__global__ void comp_out_kernel(int nu, const int32_t* __restrict__ unit_comp,
                                const uint8_t* __restrict__ status,
                                const int32_t* __restrict__ iters,
                                const int32_t* __restrict__ pstart,
                                int32_t* __restrict__ comp_iters, int32_t* __restrict__ comp_status,
                                int32_t* __restrict__ max_iters) {
  int mx = 0;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += gridDim.x * blockDim.x) {
    if (pstart[u + 1] == pstart[u]) continue;
    const int c = unit_comp ? unit_comp[u] : u;
    const int it = iters[u];
    atomicMax(comp_iters + c, it);
    if (status[u] == U_CAPPED) atomicMax(comp_status + c, 1);
    mx = max(mx, it);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_iters, mx);
}

}  // namespace mg
}  // namespace ni

// ================================================================== host

using namespace ni;
using namespace ni::mg;

namespace {

struct MgFixed {
  float *x, *r, *r2, *p, *s, *s2, *u, *w, *hw, *dinv;
  uint8_t* imask;
  int32_t *par0, *unit;
  uint16_t* slot;
  int32_t *comp_size, *nslots, *slot_base, *tile_flag, *tile_pos, *tiles, *tmp;
  int32_t *cc_parent, *cc_flag, *cc_rank, *unit_comp;
  int32_t* counters;  // [0] missing, [1] NS, [2] NA, [3] NU, [4] level n, [5] nact, [6] active,
                      // [7] max iters
  void* scan_ws;
};

void carve_fixed(Carver& c, MgFixed& f, const Geo& g, int count) {
  const int64_t npad = g.npad;
  f.x = c.take<float>(npad);
  f.r = c.take<float>(npad);
  f.r2 = c.take<float>(npad);
  f.p = c.take<float>(npad);
  f.s = c.take<float>(npad);
  f.s2 = c.take<float>(npad);
  f.u = c.take<float>(npad);
  f.w = c.take<float>(npad);
  f.hw = c.take<float>(npad);
  f.dinv = c.take<float>(npad);
  f.imask = c.take<uint8_t>(npad);
  f.par0 = c.take<int32_t>(npad);
  f.unit = c.take<int32_t>(npad);
  f.slot = c.take<uint16_t>(npad);
  f.comp_size = c.take<int32_t>(count + 1);
  f.nslots = c.take<int32_t>(g.ntiles + 1);
  f.slot_base = c.take<int32_t>(g.ntiles + 1);
  f.tile_flag = c.take<int32_t>(g.ntiles + 1);
  f.tile_pos = c.take<int32_t>(g.ntiles + 1);
  f.tiles = c.take<int32_t>(g.ntiles + 1);
  f.tmp = c.take<int32_t>(int64_t(g.ntiles) * TPX);
  f.cc_parent = c.take<int32_t>(g.npix);
  f.cc_flag = c.take<int32_t>(g.npix + 1);
  f.cc_rank = c.take<int32_t>(g.npix + 1);
  f.unit_comp = c.take<int32_t>(g.npix + 1);
  f.counters = c.take<int32_t>(16);
  const int64_t scan_n = std::max<int64_t>(std::max<int64_t>(g.npix + 1, g.ntiles + 1),
                                           int64_t(count) + 1);
  f.scan_ws = c.take<char>(scan_ws_bytes(scan_n));
}

// bytes of one coarse unknown: blk, unit, nbr[8], cond[8], dinv, parent,
// child[4], b, e + its share of the block table
constexpr int64_t kBytesPerUnknown = 4 * (2 + 8 + 8 + 1 + 1 + 4 + 4 + 2 + 8);

int64_t level_estimate(const Geo& g) {
  // ~ npix/4 * 4/3 over all levels, + boundary aggregates and block tables
  return g.npix / 2 + 65536;
}

void carve_level(Carver& c, Level& L, int n, bool children) {
  L.blk = c.take<int32_t>(n + 1);
  L.unit = c.take<int32_t>(n + 1);
  L.nbr = c.take<int32_t>(8 * int64_t(n) + 1);
  L.cond = c.take<float>(8 * int64_t(n) + 1);
  L.dinv = c.take<float>(n + 1);
  L.parent = c.take<int32_t>(n + 1);
  L.child = children ? c.take<int32_t>(4 * int64_t(n) + 1) : nullptr;
  L.b = c.take<float>(n + 1);
  L.x1 = c.take<float>(n + 1);
  L.x2 = c.take<float>(n + 1);
  L.e = c.take<float>(n + 1);
  L.lnk = c.take<Link8>(n + 1);
}

int grid_for(int64_t n, int per = 256) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, int64_t(kSMs) * 32)));
}

// Tensor maps of the padded planes for the fine passes' TMA boxes.
int make_tma_maps(TmaMaps& tm, const Geo& g, const MgFixed& f) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    NI_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return NI_ERR_CUDA;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  const cuuint64_t rows = cuuint64_t(g.rows + RM + RB);
  auto mk = [&](CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esz, int bw,
                int bh) -> int {
    const cuuint64_t dims[2] = {cuuint64_t(g.P), rows};
    const cuuint64_t strides[1] = {cuuint64_t(g.P) * esz};
    const cuuint32_t box[2] = {cuuint32_t(bw), cuuint32_t(bh)};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
      return NI_ERR_CUDA;
    }
    return NI_OK;
  };
  const auto F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  NI_TRY(mk(&tm.r[0], f.r, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.r[1], f.r2, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.s[0], f.s, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.s[1], f.s2, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.w, f.w, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.dinv, f.dinv, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.hw, f.hw, F32, 4, BW, BH1));
  NI_TRY(mk(&tm.rB[0], f.r, F32, 4, BW, BH2));
  NI_TRY(mk(&tm.rB[1], f.r2, F32, 4, BW, BH2));
  NI_TRY(mk(&tm.dinvB, f.dinv, F32, 4, BW, BH2));
  NI_TRY(mk(&tm.hwB, f.hw, F32, 4, BW, BH2));
  NI_TRY(mk(&tm.parB, f.par0, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, BW, BH2));
  NI_TRY(mk(&tm.imB, f.imask, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, BWM, BH1));
  NI_TRY(mk(&tm.uI, f.u, F32, 4, TX, TY));
  NI_TRY(mk(&tm.pI, f.p, F32, 4, TX, TY));
  NI_TRY(mk(&tm.xI, f.x, F32, 4, TX, TY));
  return NI_OK;
}

// Compact links of a built level (counters[10]: offset overflow flag) and
// its count of unknowns with a link (counters[5], written by the links
// kernel): one read-back.
int compact_level(Level& L, int32_t* counters, cudaStream_t st) {
  NI_CUDA_TRY(cudaMemsetAsync(counters + 10, 0, sizeof(int32_t), st));
  if (L.n > 0) {
    NI_COUNT_LAUNCH(), compact_links_kernel<<<grid_for(L.n), 256, 0, st>>>(L.n, L.nbr, L.cond,
                                                                          L.lnk, counters + 10);
    NI_LAUNCH_CHECK();
  }
  int32_t h[6];
  NI_CUDA_TRY(cudaMemcpyAsync(h, counters + 5, sizeof(h), cudaMemcpyDeviceToHost, st));
  NI_CUDA_TRY(cudaStreamSynchronize(st));
  L.nact = h[0];
  L.cmp = h[5] == 0 && NI_MG_CMP_LINKS;
  return NI_OK;
}

// Events of the calling thread, created once per device (not per call).
// V-cycles are enqueued kLag ahead of the last one whose outcome (active
// units, processed pixels) the host has read: per V-cycle a pinned slot and
// an event, kRing of them in a ring.
constexpr int kLag = 2, kRing = 4;
struct EventPool {
  int dev = -1;
  cudaEvent_t ev[2 + 5 * kRing + kRing];  // loop; per ring slot: 5 stage marks; slot done
  int32_t* host = nullptr;                 // pinned [kRing][4]
};
thread_local EventPool g_events;

int thread_events(cudaEvent_t** out) {
  int dev = 0;
  NI_CUDA_TRY(cudaGetDevice(&dev));
  if (g_events.dev != dev) {
    if (g_events.dev >= 0)
      for (cudaEvent_t e : g_events.ev) cudaEventDestroy(e);
    g_events.dev = -1;
    for (cudaEvent_t& e : g_events.ev) NI_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDefault));
    if (!g_events.host)
      NI_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&g_events.host),
                                sizeof(int32_t) * 4 * kRing, cudaHostAllocPortable));
    g_events.dev = dev;
  }
  *out = g_events.ev;
  return NI_OK;
}

}  // namespace

extern "C" int ni_fill_mg_workspace_size(int B, int H, int W, int connectivity, int count,
                                         size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  const Geo g = make_geo(B, H, W);
  Sizer s;
  MgFixed f;
  carve_fixed(s, f, g, count);
  // slot / unit arrays (estimates; ni_fill_mg reports the exact need)
  const int64_t ns = int64_t(g.ntiles) * 4 + 1024;
  s.take<int32_t>(ns * 4);
  s.take<double>(ns * 3);
  s.take<char>(int64_t(count + 1) * 64);
  s.take<char>(level_estimate(g) * kBytesPerUnknown + g.npix * 2 + (1 << 20));
  *bytes = s.used;
  return NI_OK;
}

extern "C" int ni_fill_mg(const int32_t* labels, int count, const double* omega_a,
                          const double* omega_b, const double* gamma, const uint8_t* eflags,
                          int B, int H, int W, int connectivity, int model, double cg_tol,
                          int cg_max_iters, double* z_out, int32_t* comp_iters,
                          int32_t* comp_status, void* workspace, size_t workspace_bytes,
                          size_t* needed_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(model == 0 || (model == 1 && connectivity == 4), "bad model/connectivity");
  NI_CHECK_ARG(cg_tol > 0, "cg_tol must be positive");
  NI_CHECK_ARG(count >= 0, "count must be non-negative");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo g = make_geo(B, H, W);
  Carver cv(workspace, workspace_bytes);
  MgFixed f;
  carve_fixed(cv, f, g, count);
  auto too_small = [&](size_t extra) {
    if (needed_bytes) *needed_bytes = cv.used + extra;
    set_error("ni_fill_mg: workspace too small (%zu < %zu)", workspace_bytes, cv.used + extra);
    return NI_ERR_WORKSPACE;
  };
  if (!workspace || !cv.ok())
    return too_small(size_t(level_estimate(g) * kBytesPerUnknown + g.npix * 2));
  cudaEvent_t* ev = nullptr;  // [0], [1]: the PCG loop; [2..6]: one V-cycle's stages
  NI_TRY(thread_events(&ev));
  const cudaEvent_t e0 = ev[0], e1 = ev[1];
  const bool prof = g_fill_profile != 0;
  double stage_ms[4] = {0.0, 0.0, 0.0, 0.0};
  long long px_vcycles = 0;
  const int npb = grid_for(g.npix);
  const size_t npad = size_t(g.npad);
  // ---- fine planes
  for (float* pl : {f.x, f.r, f.r2, f.p, f.s, f.s2, f.u, f.w, f.hw, f.dinv})
    NI_CUDA_TRY(cudaMemsetAsync(pl, 0, npad * sizeof(float), st));
  NI_CUDA_TRY(cudaMemsetAsync(f.imask, 0, npad, st));
  NI_CUDA_TRY(cudaMemsetAsync(f.par0, 0xff, npad * sizeof(int32_t), st));
  NI_CUDA_TRY(cudaMemsetAsync(f.unit, 0xff, npad * sizeof(int32_t), st));
  NI_CUDA_TRY(cudaMemsetAsync(f.slot, 0xff, npad * sizeof(uint16_t), st));
  NI_CUDA_TRY(cudaMemsetAsync(f.comp_size, 0, sizeof(int32_t) * (count + 1), st));
  NI_CUDA_TRY(cudaMemsetAsync(f.counters, 0, sizeof(int32_t) * 16, st));
#define NI_MG_PREP(CONN, MODEL)                                                                  \
  NI_COUNT_LAUNCH(), prep_kernel<CONN, MODEL><<<dim3(div_up(W, 32), div_up(int64_t(B) * H, 8)), 256, 0, st>>>( \
                         labels, omega_a, omega_b, gamma, eflags, H, W, g.P, g.npix, f.hw, f.r, \
                         f.imask, f.dinv, f.comp_size, f.counters + 0)
  if (connectivity == 8) NI_MG_PREP(8, 0);
  else if (model == 0) NI_MG_PREP(4, 0);
  else NI_MG_PREP(4, 1);
#undef NI_MG_PREP
  NI_LAUNCH_CHECK();
  // Host-only set-up of the fine passes (opt-in shared-memory sizes once per
  // process, the 16 tensor maps of this call's planes: ~0.3 ms of driver
  // calls), done here while the GPU runs prep_kernel instead of between the
  // hierarchy build and the first pass A.
  {
    static std::atomic<bool> attrs_set{false};
    if (!attrs_set.load(std::memory_order_acquire)) {
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_b_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassBSmem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_b_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassBSmem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_a_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassASmem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_a_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassASmem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_b2_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassB2Smem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_b2_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassB2Smem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_a2_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassA2Smem)));
      NI_CUDA_TRY(cudaFuncSetAttribute(pass_a2_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kPassA2Smem)));
      attrs_set.store(true, std::memory_order_release);
    }
  }
  TmaMaps tm;
  memset(&tm, 0, sizeof(tm));
  NI_TRY(make_tma_maps(tm, g, f));
  int32_t hc[16];
  NI_CUDA_TRY(cudaMemcpyAsync(hc, f.counters, sizeof(hc), cudaMemcpyDeviceToHost, st));
  NI_CUDA_TRY(cudaStreamSynchronize(st));
  // ---- solve units
  int NU = count;
  const int32_t* unit_comp = nullptr;
  if (hc[0] == 0) {
    NI_COUNT_LAUNCH(), unit_from_label_kernel<<<npb, 256, 0, st>>>(labels, H, W, g.P, g.npix,
                                                                  f.imask, f.unit);
    NI_LAUNCH_CHECK();
  } else {
    NI_COUNT_LAUNCH(), cc_init_kernel<<<npb, 256, 0, st>>>(W, g.P, g.npix, f.imask, f.cc_parent);
    NI_LAUNCH_CHECK();
    if (connectivity == 8)
      NI_COUNT_LAUNCH(), cc_union_kernel<8><<<npb, 256, 0, st>>>(W, g.P, g.npix, f.imask, f.cc_parent);
    else
      NI_COUNT_LAUNCH(), cc_union_kernel<4><<<npb, 256, 0, st>>>(W, g.P, g.npix, f.imask, f.cc_parent);
    NI_LAUNCH_CHECK();
    NI_COUNT_LAUNCH(), cc_flatten_kernel<<<npb, 256, 0, st>>>(g.npix, f.cc_parent, f.cc_flag);
    NI_LAUNCH_CHECK();
    NI_TRY(exclusive_scan_i32(f.cc_flag, f.cc_rank, g.npix, f.counters + 3, f.scan_ws, st));
    NI_COUNT_LAUNCH(), cc_label_kernel<<<npb, 256, 0, st>>>(labels, W, g.P, g.npix, f.cc_parent,
                                                           f.cc_rank, f.unit, f.unit_comp);
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemcpyAsync(&NU, f.counters + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    NI_CUDA_TRY(cudaStreamSynchronize(st));
    unit_comp = f.unit_comp;
  }
  // ---- tile plan (the scans run over n + 1 entries: the last count is 0)
  NI_CUDA_TRY(cudaMemsetAsync(f.nslots + g.ntiles, 0, sizeof(int32_t), st));
  NI_COUNT_LAUNCH(), plan_tile_kernel<<<g.ntiles, NT, 0, st>>>(H, W, g.P, g.nTX, g.nTY, f.unit,
                                                              f.slot, f.nslots, f.tmp);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(f.nslots, f.slot_base, g.ntiles + 1, f.counters + 1, f.scan_ws, st));
  NI_CUDA_TRY(cudaMemcpyAsync(hc + 1, f.counters + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  NI_CUDA_TRY(cudaStreamSynchronize(st));
  const int NS = hc[1];
  // slot / unit arrays
  int32_t* slot_unit = cv.take<int32_t>(NS + 1);
  int32_t* slot_idx = cv.take<int32_t>(NS + 1);
  int32_t* skeys = cv.take<int32_t>(NS + 1);
  int32_t* plist = cv.take<int32_t>(NS + 1);
  double* partial = cv.take<double>(NPART * int64_t(NS) + NPART);
  int32_t* pstart = cv.take<int32_t>(NU + 2);
  uint8_t* ustatus = cv.take<uint8_t>(NU + 1);
  uint8_t* uupd = cv.take<uint8_t>(NU + 1);
  int32_t* uiters = cv.take<int32_t>(NU + 1);
  int32_t* ucap = cv.take<int32_t>(NU + 1);
  double* utol2 = cv.take<double>(NU + 1);
  double* ugprev = cv.take<double>(NU + 1);
  double* uaprev = cv.take<double>(NU + 1);
  double* umean = cv.take<double>(NU + 1);
  float* ualpha = cv.take<float>(NU + 1);
  float* ubeta = cv.take<float>(NU + 1);
  float* uumean = cv.take<float>(NU + 1);
  double* unit_n = cv.take<double>(NU + 1);
  size_t sort_bytes = 0;
  NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int32_t*)nullptr,
                                              (int32_t*)nullptr, (const int32_t*)nullptr,
                                              (int32_t*)nullptr, std::max(NS, 1)));
  void* sort_ws = cv.take<char>(sort_bytes + 256);
  if (!cv.ok())
    return too_small(size_t(level_estimate(g) * kBytesPerUnknown + g.npix * 2));
  NI_COUNT_LAUNCH(), plan_copy_kernel<<<g.ntiles, 128, 0, st>>>(g.ntiles, f.nslots, f.slot_base,
                                                               f.tmp, slot_unit, f.tile_flag);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(f.tile_flag, f.tile_pos, g.ntiles, f.counters + 2, f.scan_ws, st));
  NI_COUNT_LAUNCH(), tile_list_kernel<<<grid_for(g.ntiles), 256, 0, st>>>(g.ntiles, f.tile_flag,
                                                                         f.tile_pos, f.tiles);
  NI_LAUNCH_CHECK();
  if (NS > 0) {
    NI_COUNT_LAUNCH(), iota_kernel<<<grid_for(NS), 256, 0, st>>>(slot_idx, NS);
    NI_LAUNCH_CHECK();
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= NU) ++end_bit;
    size_t sb = sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(sort_ws, sb, slot_unit, skeys, slot_idx, plist,
                                                NS, 0, end_bit, st));
  }
  NI_COUNT_LAUNCH(), unit_bounds_kernel<<<grid_for(NU + 1), 256, 0, st>>>(skeys, NS, NU, pstart);
  NI_LAUNCH_CHECK();
  if (NU > 0) {
    NI_COUNT_LAUNCH(), unit_init_kernel<<<grid_for(NU), 256, 0, st>>>(
                           NU, unit_comp, f.comp_size, pstart, cg_max_iters, ustatus, uupd,
                           uiters, ucap, ualpha, ubeta);
    NI_LAUNCH_CHECK();
  }
  NI_CUDA_TRY(cudaMemcpyAsync(hc + 2, f.counters + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  NI_CUDA_TRY(cudaStreamSynchronize(st));
  const int NA = hc[2];
  // ---- hierarchy
  Level lev[MAXLEV + 1];
  int L = 0;
  if (NA > 0) {
    Level& L1 = lev[1];
    L1.Hb = div_up(H, 2);
    L1.Wb = div_up(W, 2);
    L1.nblk = int64_t(B) * L1.Hb * L1.Wb;
    L1.bstart = cv.take<int32_t>(L1.nblk + 1);
    L1.cnt = cv.take<int32_t>(L1.nblk + 1);
    if (!cv.ok()) return too_small(size_t(level_estimate(g) * kBytesPerUnknown));
    NI_CUDA_TRY(cudaMemsetAsync(L1.cnt + L1.nblk, 0, sizeof(int32_t), st));
    NI_COUNT_LAUNCH(), l1_count_kernel<<<grid_for(L1.nblk), 256, 0, st>>>(B, H, W, g.P, L1.Hb,
                                                                         L1.Wb, f.unit, L1.cnt);
    NI_LAUNCH_CHECK();
    NI_TRY(exclusive_scan_i32(L1.cnt, L1.bstart, L1.nblk + 1, f.counters + 4, f.scan_ws, st));
    NI_CUDA_TRY(cudaMemcpyAsync(&L1.n, f.counters + 4, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    NI_CUDA_TRY(cudaStreamSynchronize(st));
    carve_level(cv, L1, L1.n, false);
    if (!cv.ok()) return too_small(size_t(level_estimate(g) * kBytesPerUnknown));
    NI_CUDA_TRY(cudaMemsetAsync(L1.x2, 0, sizeof(float) * (L1.n + 1), st));
    NI_COUNT_LAUNCH(), l1_assign_kernel<<<grid_for(L1.nblk), 256, 0, st>>>(
                           B, H, W, g.P, L1.Hb, L1.Wb, f.unit, L1.bstart, L1.blk, L1.unit, f.par0);
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemsetAsync(L1.parent, 0xff, sizeof(int32_t) * (L1.n + 1), st));
    NI_CUDA_TRY(cudaMemsetAsync(f.counters + 5, 0, sizeof(int32_t), st));
    if (connectivity == 8)
      NI_COUNT_LAUNCH(), l1_links_kernel<8><<<grid_for(L1.n), 256, 0, st>>>(
                             L1.n, H, W, g.P, L1.Hb, L1.Wb, L1.bstart, L1.blk, L1.unit, f.unit,
                             f.hw, f.imask, L1.nbr, L1.cond, L1.dinv, f.counters + 5);
    else
      NI_COUNT_LAUNCH(), l1_links_kernel<4><<<grid_for(L1.n), 256, 0, st>>>(
                             L1.n, H, W, g.P, L1.Hb, L1.Wb, L1.bstart, L1.blk, L1.unit, f.unit,
                             f.hw, f.imask, L1.nbr, L1.cond, L1.dinv, f.counters + 5);
    NI_LAUNCH_CHECK();
    NI_TRY(compact_level(L1, f.counters, st));
    L = 1;
    while (L < MAXLEV && lev[L].nact > 0) {
      Level& C = lev[L];
      Level& N = lev[L + 1];
      N.Hb = div_up(C.Hb, 2);
      N.Wb = div_up(C.Wb, 2);
      N.nblk = int64_t(B) * N.Hb * N.Wb;
      N.bstart = cv.take<int32_t>(N.nblk + 1);
      N.cnt = cv.take<int32_t>(N.nblk + 1);
      if (!cv.ok()) return too_small(size_t(C.n) * kBytesPerUnknown * 2);
      NI_CUDA_TRY(cudaMemsetAsync(N.cnt + N.nblk, 0, sizeof(int32_t), st));
      NI_COUNT_LAUNCH(), lc_count_kernel<<<grid_for(N.nblk), 256, 0, st>>>(
                             N.nblk, N.Hb, N.Wb, C.Hb, C.Wb, C.bstart, C.unit, C.dinv, N.cnt);
      NI_LAUNCH_CHECK();
      NI_TRY(exclusive_scan_i32(N.cnt, N.bstart, N.nblk + 1, f.counters + 4, f.scan_ws, st));
      NI_CUDA_TRY(cudaMemcpyAsync(&N.n, f.counters + 4, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      NI_CUDA_TRY(cudaStreamSynchronize(st));
      if (N.n == 0) break;
      carve_level(cv, N, N.n, true);
      if (!cv.ok()) return too_small(size_t(N.n) * kBytesPerUnknown * 2);
      NI_CUDA_TRY(cudaMemsetAsync(N.x2, 0, sizeof(float) * (N.n + 1), st));
      NI_COUNT_LAUNCH(), lc_assign_kernel<<<grid_for(N.nblk), 256, 0, st>>>(
                             N.nblk, N.Hb, N.Wb, C.Hb, C.Wb, C.bstart, C.unit, C.dinv, N.bstart,
                             N.n, N.blk, N.unit, N.child, C.parent);
      NI_LAUNCH_CHECK();
      NI_CUDA_TRY(cudaMemsetAsync(N.parent, 0xff, sizeof(int32_t) * (N.n + 1), st));
      NI_CUDA_TRY(cudaMemsetAsync(f.counters + 5, 0, sizeof(int32_t), st));
      NI_COUNT_LAUNCH(), lc_links_kernel<<<grid_for(N.n), 256, 0, st>>>(
                             N.n, N.Hb, N.Wb, N.bstart, N.blk, N.unit, N.child, C.n, C.nbr,
                             C.cond, C.parent, N.nbr, N.cond, N.dinv, f.counters + 5);
      NI_LAUNCH_CHECK();
      NI_TRY(compact_level(N, f.counters, st));
      ++L;
    }
    // the coarsest level used is the last one with a link
    while (L > 1 && lev[L].nact == 0) --L;
  }
  if (needed_bytes) *needed_bytes = cv.used;
  // ---- PCG
  FineArgs fa;
  fa.H = H;
  fa.W = W;
  fa.P = g.P;
  fa.nTX = g.nTX;
  fa.nTY = g.nTY;
  fa.tiles = f.tiles;
  fa.x = f.x;
  fa.par = 0;
  fa.rbuf[0] = f.r;
  fa.rbuf[1] = f.r2;
  fa.sbuf[0] = f.s;
  fa.sbuf[1] = f.s2;
  fa.p = f.p;
  fa.u = f.u;
  fa.w = f.w;
  fa.hw = f.hw;
  fa.dinv = f.dinv;
  fa.imask = f.imask;
  fa.par0 = f.par0;
  fa.unit = f.unit;
  fa.slot = f.slot;
  fa.slot_base = f.slot_base;
  fa.slot_unit = slot_unit;
  fa.status = ustatus;
  fa.upd = uupd;
  fa.alpha = ualpha;
  fa.beta = ubeta;
  fa.b1 = lev[1].b;
  fa.x1_1 = lev[1].x1;
  fa.dinv1 = lev[1].dinv;
  fa.e1 = lev[1].e;
  fa.partial = partial;
  fa.umean = uumean;
  if (NA > 0) {  // pixels per unit (x = 0 here: the sums are the counts)
    NI_CUDA_TRY(cudaMemsetAsync(uumean, 0, sizeof(float) * (NU + 1), st));
    NI_COUNT_LAUNCH(), xsum_kernel<<<NA, NT, 0, st>>>(fa);
    NI_LAUNCH_CHECK();
    NI_COUNT_LAUNCH(), unit_mean_kernel<<<grid_for(int64_t(NU) * 32), 256, 0, st>>>(
                           NU, pstart, plist, partial, umean, unit_n);
    NI_LAUNCH_CHECK();
  }
  ScalarArgs sa;
  sa.nu = NU;
  sa.pstart = pstart;
  sa.plist = plist;
  sa.partial = partial;
  sa.unit_n = unit_n;
  sa.umean = uumean;
  sa.rtol = cg_tol;
  sa.status = ustatus;
  sa.upd = uupd;
  sa.iters = uiters;
  sa.cap = ucap;
  sa.tol2 = utol2;
  sa.gprev = ugprev;
  sa.aprev = uaprev;
  sa.alpha = ualpha;
  sa.beta = ubeta;
  sa.nactive = f.counters + 6;
  sa.px_done = reinterpret_cast<unsigned long long*>(f.counters + 8);
  {
    const char* tr = NI_ENV_ONCE("NI_MG_TRACE");
    sa.trace_unit = tr ? atoi(tr) : -1;
  }
  int vcycles = 0;
  // ---- the coarse part of one V-cycle (levels 1..L), between pass A (which
  // leaves b and x1 = OM dinv b on level 1) and pass B (which prolongs e of
  // level 1).  Levels >= 2 run kCoarseSweeps damped-Jacobi sweeps before and
  // after their coarse correction instead of one: they hold 1/16, 1/64, ... of
  // the pixels, so the extra sweeps are cheap, and the PCG needs a quarter
  // fewer V-cycles (scripts/mg_blueprint.py, MG_NU=2 MG_NU_FROM=2: 12.5 -> 9.2;
  // a third sweep gains nothing more).  Any number of sweeps keeps the
  // preconditioner symmetric positive definite.  (A W-cycle over levels 2-3
  // needed 8.0 but its two-visit operator 2M - MAM is indefinite wherever the
  // 1.9x over-corrected M has an eigenvalue of AM above 2: on the 4096^2 map
  // the PCG then broke down and left a 6e-3 error in the fill.)
  int nu2 = 2;
  {
    const char* a = NI_ENV_ONCE("NI_MG_COARSE_SWEEPS");
    if (a) nu2 = atoi(a) >= 2 ? 2 : 1;
  }
  // the pre-smoothed state of level l: x1 after one sweep, e (free on levels
  // >= 2) after two
  auto xpre = [&](int l) -> float* { return (l >= 2 && nu2 == 2) ? lev[l].e : lev[l].x1; };
  auto launch_down = [&](int l) -> int {  // b, x1 of level l + 1 from level l
    const Level& C = lev[l];
    const Level& N = lev[l + 1];
    if (C.cmp)
      NI_COUNT_LAUNCH(), down_kernel<true><<<grid_for(N.n), 256, 0, st>>>(
                             N.n, N.child, C.n, C.nbr, C.cond, C.lnk, xpre(l), C.b, N.dinv, N.b,
                             N.x1, N.unit, ustatus);
    else
      NI_COUNT_LAUNCH(), down_kernel<false><<<grid_for(N.n), 256, 0, st>>>(
                             N.n, N.child, C.n, C.nbr, C.cond, C.lnk, xpre(l), C.b, N.dinv, N.b,
                             N.x1, N.unit, ustatus);
    NI_LAUNCH_CHECK();
    return NI_OK;
  };
  // one damped-Jacobi sweep of level l from xs: out = xs + OM dinv (b - A xs);
  // scatter: hand x2 = xpre + OC out to the children instead of storing it
  auto launch_sweep = [&](int l, const float* xs, float* out, bool scatter) -> int {
    const Level& C = lev[l];
#define NI_MG_UP(SC, CM, EOUT, CH, X1C, X2C, NC)                                               \
  NI_COUNT_LAUNCH(), up_kernel<SC, CM><<<grid_for(C.n), 256, 0, st>>>(                           \
                         C.n, C.nbr, C.cond, C.lnk, C.dinv, C.b, xs, EOUT, CH, X1C, X2C, NC, C.unit, \
                         ustatus)
    if (scatter) {
      if (C.cmp) NI_MG_UP(true, true, nullptr, C.child, xpre(l - 1), lev[l - 1].x2, lev[l - 1].n);
      else NI_MG_UP(true, false, nullptr, C.child, xpre(l - 1), lev[l - 1].x2, lev[l - 1].n);
    } else {
      if (C.cmp) NI_MG_UP(false, true, out, nullptr, nullptr, nullptr, 0);
      else NI_MG_UP(false, false, out, nullptr, nullptr, nullptr, 0);
    }
#undef NI_MG_UP
    NI_LAUNCH_CHECK();
    return NI_OK;
  };
  // the first level of the single-launch tail (L + 1: none)
  int T = L + 1;
  TailArgs ta;
  memset(&ta, 0, sizeof(ta));
  {
    const char* a = NI_ENV_ONCE("NI_MG_TAIL");
    const bool on = !a || atoi(a) != 0;
    int t0 = 2;
    while (t0 <= L && lev[t0].n > kTailMaxN) ++t0;
    bool ok = on && t0 <= L && L - t0 + 1 <= kTailMaxLevels;
    for (int l = t0; ok && l <= L; ++l) ok = lev[l].cmp;
    if (ok) {
      T = t0;
      ta.nlev = L - T + 1;
      ta.nu2 = nu2;
      for (int l = T - 1; l <= L; ++l) {
        TailLevel& V = ta.lv[l - (T - 1)];
        V.n = lev[l].n;
        V.lnk = lev[l].lnk;
        V.dinv = lev[l].dinv;
        V.child = lev[l].child;
        V.b = lev[l].b;
        V.x1 = lev[l].x1;
        V.x2 = lev[l].x2;
        V.e = lev[l].e;
      }
      ta.xpre0 = xpre(T - 1);
      // the tail does not skip the unknowns of units that never become active
      // (zero right-hand side): give them defined values (b, x1, x2, e are
      // carved back to back)
      for (int l = T; l <= L; ++l)
        NI_CUDA_TRY(cudaMemsetAsync(lev[l].b, 0,
                                    size_t(reinterpret_cast<char*>(lev[l].e + lev[l].n + 1) -
                                           reinterpret_cast<char*>(lev[l].b)), st));
    }
  }
  auto coarse_cycle = [&]() -> int {
    for (int l = 1; l < T; ++l) {
      if (l >= 2 && nu2 == 2) NI_TRY(launch_sweep(l, lev[l].x1, lev[l].e, false));  // second pre-sweep
      if (l < L) NI_TRY(launch_down(l));
    }
    if (T <= L) {  // levels T..L and back, leaving x2 of level T - 1
      NI_COUNT_LAUNCH(), tail_kernel<<<1, kTailThreads, 0, st>>>(ta);
      NI_LAUNCH_CHECK();
    }
    for (int l = std::min(L, T - 1); l >= 2; --l) {
      const float* xs = l == L ? xpre(l) : lev[l].x2;
      if (nu2 == 2) {  // first post-sweep into x1 (free once x2 exists)
        NI_TRY(launch_sweep(l, xs, lev[l].x1, false));
        xs = lev[l].x1;
      }
      NI_TRY(launch_sweep(l, xs, nullptr, true));
    }
    NI_TRY(launch_sweep(1, L == 1 ? lev[1].x1 : lev[1].x2, lev[1].e, false));
    return NI_OK;
  };
  NI_CUDA_TRY(cudaEventRecord(e0, st));
  if (NA > 0) {
    int32_t* hslot = g_events.host;
    // outcome of V-cycle j: nact = 0 means every unit is done; V-cycles
    // enqueued after it find nothing to do (tiles and unknowns of finished
    // units are skipped)
    auto settle = [&](int j, bool& fin) -> int {
      const int r = j % kRing;
      NI_CUDA_TRY(cudaEventSynchronize(ev[2 + 5 * kRing + r]));
      const int32_t* hv = hslot + 4 * r;
      if (prof) {
        unsigned long long pxd;
        memcpy(&pxd, hv + 2, sizeof(pxd));
        px_vcycles += (long long)pxd;
        for (int k = 0; k < 4; ++k) {
          float t = 0.f;
          NI_CUDA_TRY(cudaEventElapsedTime(&t, ev[2 + 5 * r + k], ev[2 + 5 * r + k + 1]));
          stage_ms[k] += t;
        }
      }
      fin = hv[0] == 0;
      return NI_OK;
    };
    int done_at = -1;  // the V-cycle after which no unit was active
    for (int it = 0;; ++it) {
      if (it >= kLag) {
        bool fin = false;
        NI_TRY(settle(it - kLag, fin));
        if (fin) {
          done_at = it - kLag;
          break;
        }
      }
      cudaEvent_t* evs = ev + 2 + 5 * (it % kRing);
      if (prof) NI_CUDA_TRY(cudaEventRecord(evs[0], st));
#if NI_MG_V2
      if (connectivity == 8) NI_COUNT_LAUNCH(), pass_a2_kernel<8><<<NA, NT, kPassA2Smem, st>>>(fa, tm);
      else NI_COUNT_LAUNCH(), pass_a2_kernel<4><<<NA, NT, kPassA2Smem, st>>>(fa, tm);
#else
      if (connectivity == 8) NI_COUNT_LAUNCH(), pass_a_kernel<8><<<NA, NT, kPassASmem, st>>>(fa, tm);
      else NI_COUNT_LAUNCH(), pass_a_kernel<4><<<NA, NT, kPassASmem, st>>>(fa, tm);
#endif
      fa.par ^= 1;  // pass B and the next pass A read the r / s pass A wrote
      NI_LAUNCH_CHECK();
      if (prof) NI_CUDA_TRY(cudaEventRecord(evs[1], st));
      NI_TRY(coarse_cycle());
      if (prof) NI_CUDA_TRY(cudaEventRecord(evs[2], st));
#if NI_MG_V2 && NI_MG_B_V2
      if (connectivity == 8) NI_COUNT_LAUNCH(), pass_b2_kernel<8><<<NA, NT, kPassB2Smem, st>>>(fa, tm);
      else NI_COUNT_LAUNCH(), pass_b2_kernel<4><<<NA, NT, kPassB2Smem, st>>>(fa, tm);
#else
      if (connectivity == 8) NI_COUNT_LAUNCH(), pass_b_kernel<8><<<NA, NT, kPassBSmem, st>>>(fa, tm);
      else NI_COUNT_LAUNCH(), pass_b_kernel<4><<<NA, NT, kPassBSmem, st>>>(fa, tm);
#endif
      NI_LAUNCH_CHECK();
      if (prof) NI_CUDA_TRY(cudaEventRecord(evs[3], st));
      // counters [6] active units, [8..9] processed unit pixels (u64)
      NI_CUDA_TRY(cudaMemsetAsync(f.counters + 6, 0, 4 * sizeof(int32_t), st));
      NI_COUNT_LAUNCH(), scalar_kernel<<<grid_for(int64_t(NU) * 32), 256, 0, st>>>(sa);
      NI_LAUNCH_CHECK();
      if (prof) NI_CUDA_TRY(cudaEventRecord(evs[4], st));
      NI_CUDA_TRY(cudaMemcpyAsync(hslot + 4 * (it % kRing), f.counters + 6, 4 * sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, st));
      NI_CUDA_TRY(cudaEventRecord(ev[2 + 5 * kRing + it % kRing], st));
    }
    // the V-cycles still in flight after done_at are no-ops; settle them so
    // the ring and the profile are consistent
    for (int j = done_at + 1; j < done_at + 1 + kLag; ++j) {
      bool fin = false;
      NI_TRY(settle(j, fin));
    }
    vcycles = done_at + 1;
  }
  NI_CUDA_TRY(cudaEventRecord(e1, st));
  // ---- output: x minus its per-unit mean
  if (NA > 0) {
    NI_COUNT_LAUNCH(), xsum_kernel<<<NA, NT, 0, st>>>(fa);
    NI_LAUNCH_CHECK();
    NI_COUNT_LAUNCH(), unit_mean_kernel<<<grid_for(int64_t(NU) * 32), 256, 0, st>>>(
                           NU, pstart, plist, partial, umean, nullptr);
    NI_LAUNCH_CHECK();
  }
  NI_COUNT_LAUNCH(), output_kernel<<<npb, 256, 0, st>>>(W, g.P, g.npix, f.x, f.unit, umean, z_out);
  NI_LAUNCH_CHECK();
  NI_CUDA_TRY(cudaMemsetAsync(comp_iters, 0, sizeof(int32_t) * std::max(count, 1), st));
  NI_CUDA_TRY(cudaMemsetAsync(comp_status, 0, sizeof(int32_t) * std::max(count, 1), st));
  NI_CUDA_TRY(cudaMemsetAsync(f.counters + 7, 0, sizeof(int32_t), st));
  if (NU > 0) {
    NI_COUNT_LAUNCH(), comp_out_kernel<<<grid_for(NU), 256, 0, st>>>(
                           NU, unit_comp, ustatus, uiters, pstart, comp_iters, comp_status,
                           f.counters + 7);
    NI_LAUNCH_CHECK();
  }
  int32_t mx = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&mx, f.counters + 7, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  NI_CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  NI_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  FillReport& rep = g_fill_report;
  rep.cg_ms = ms;
  rep.px_iters = 0;
  rep.max_iters = mx;
  rep.grid = NA;
  rep.ntiles = g.ntiles;
  rep.npartials = NS;
  rep.mg_levels = L;
  rep.mg_vcycles = vcycles;
  for (int k = 0; k < 4; ++k) rep.mg_ms[k] = prof ? stage_ms[k] : 0.0;
  rep.mg_px_vcycles = prof ? px_vcycles : 0;
  for (int l = 0; l < 16; ++l) rep.mg_n[l] = l >= 1 && l <= L ? lev[l].n : 0;
  return NI_OK;
}

// K3 -- fill_components (solver.py:195-239) as ONE batched CG over every
// component of the partition, matrix-free on the pixel grid.
//
// Per component c the reference solves (A^T W A) x = A^T W b with scipy's
// unpreconditioned CG (x0 = 0, stop when ||r|| < rtol ||b|| at the top of an
// iteration, cap max(cg_max_iters, n_c); solver.py:97-122).  At the fill
// state z = 0 every bilateral factor is 1/2 (continuity.py:302-308), so
// W_a = gamma_a^2 / 2 and A^T W A is the graph Laplacian of the intra-
// component valid edges with conductance c_ab = W_a + W_b (SURVEY.md
// Appendix A).  All components are iterated together; each keeps its own
// alpha/beta/rho, stop test and cap, exactly as separate scipy solves would.
//
// Data layout in HBM (per pixel, npix = B*H*W, row-major):
//   x, r, p, q : float32 CG vectors
//   hw         : float32 W_a = gamma_a^2 / 2 (conductance c_ab = hw_a + hw_b)
//   imask      : uint8 stencil mask, bit k = forward edge k intra-component
//                and valid, bit 4+k = backward edge k (pixel - offset_k)
//   slot       : uint8 index of the pixel's component inside its tile
//                (0xFF = singleton / invalid)
// Tiles are 32 x 8 pixels (one warp per row).  Each tile owns one partial-sum
// slot per component it touches; a component's dot products are the sum of
// its slots' partials in tile order (static plan => bit-reproducible, no
// floating-point atomics).  The last CTA of a component to finish a sweep
// (integer arrival counter) reduces its partials and updates its scalars,
// so each CG iteration is exactly two kernel launches:
//   sweep 1: p = r + beta p ; q = A p ; <p,q>   -> alpha
//   sweep 2: x += alpha p ; r -= alpha q ; <r,r> -> stop test, beta
// Algorithmic bytes per active pixel and iteration (8-connectivity):
//   sweep 1 reads r, p, hw (+ halo from L2), imask, slot; writes p, q
//   sweep 2 reads x, r, p, q, slot; writes x, r
//   => 4*3+1+1 + 8  +  4*4+1 + 8  = 46 B/px (independent of connectivity).
#include <cub/device/device_radix_sort.cuh>

#include "ni_common.cuh"

namespace ni {

constexpr int TX = 32, TY = 8, TPX = TX * TY;
constexpr uint8_t kNoSlot = 0xFF;

enum : uint8_t { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_CAPPED = 2, ST_IDLE = 3 };

struct FillState {
  double* rho;
  double* alpha;
  double* beta;
  double* tol;
  int32_t* iters;
  int32_t* cap;
  uint8_t* status;
  int32_t* active;  // number of active components
};

struct Plan {
  int ntx, nty;                // tiles per row / column
  const int32_t* slot_base;    // [ntiles] first partial of the tile
  const int32_t* nslots;       // [ntiles]
  const int32_t* partial_comp; // [P] component of each partial
  const int32_t* comp_pstart;  // [C+1] partial range per component (sorted)
  const int32_t* comp_plist;   // [P] partial indices grouped by component
  int32_t* comp_cnt;           // [C] arrival counters (zero between sweeps)
  double* partial;             // [P]
};

// ----------------------------------------------------------------- setup

template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) prep_kernel(
    const int32_t* __restrict__ labels, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int64_t npix, float* __restrict__ hw,
    uint8_t* __restrict__ imask, float* __restrict__ x, float* __restrict__ r,
    float* __restrict__ p, float* __restrict__ q, int32_t* __restrict__ comp_size) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t lab = labels[i];
    x[i] = 0.f;
    p[i] = 0.f;
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
      // forward edge (i -> j): row centred at i is the "a" row
      if ((ef >> k) & (ef >> (4 + k)) & 1) {
        const int64_t j = i + int64_t(dv) * W + du;
        if (labels[j] == lab) {
          m |= uint8_t(1u << k);
          const double wb = 0.5 * (gamma[j] * gamma[j]);
          const double oa = omega_a[k * npix + i];
          const double ob = MODEL == 0 ? -oa : omega_b[k * npix + i];
          b += wa * oa - wb * ob;  // solver.py:83-93 row 2i and 2i+1 via A^T W b
        }
      }
      // backward edge (j -> i) with j = i - offset_k: i is the "b" endpoint
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

// One CTA per tile: the tile's distinct multi-pixel components, ascending.
__global__ void __launch_bounds__(TPX) tile_slots_kernel(const int32_t* __restrict__ labels,
                                                         const int32_t* __restrict__ comp_size,
                                                         int rows, int W, int ntx,
                                                         int32_t* __restrict__ nslots,
                                                         int32_t* __restrict__ tile_labels,
                                                         uint8_t* __restrict__ slot) {
  __shared__ int32_t key[TPX];
  __shared__ int32_t uniq[TPX];
  __shared__ int32_t nuniq;
  const int tile = blockIdx.x;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int gx = (tile % ntx) * TX + tx, gy = (tile / ntx) * TY + ty;
  const bool in = gx < W && gy < rows;
  const int64_t i = int64_t(gy) * W + gx;
  int32_t lab = in ? labels[i] : -1;
  if (lab >= 0 && comp_size[lab] < 2) lab = -1;  // singletons never iterate (solver.py:220)
  const int tid = threadIdx.x;
  key[tid] = lab < 0 ? INT32_MAX : lab;
  __syncthreads();
  // bitonic sort of 256 keys
  for (int k = 2; k <= TPX; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      int ixj = tid ^ j;
      if (ixj > tid) {
        int32_t a = key[tid], b = key[ixj];
        bool up = (tid & k) == 0;
        if ((a > b) == up) {
          key[tid] = b;
          key[ixj] = a;
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) nuniq = 0;
  __syncthreads();
  // unique (ordered): position of each first occurrence via warp-serial scan
  const bool first = key[tid] != INT32_MAX && (tid == 0 || key[tid - 1] != key[tid]);
  // prefix count of "first" flags (block scan over 256 via warp ballots)
  const unsigned bal = __ballot_sync(0xffffffffu, first);
  __shared__ int32_t wcount[TPX / 32];
  if ((tid & 31) == 0) wcount[tid >> 5] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < (tid >> 5); ++w) before += wcount[w];
  before += __popc(bal & ((1u << (tid & 31)) - 1));
  if (first) uniq[before] = key[tid];
  if (tid == TPX - 1) {
    int tot = 0;
    for (int w = 0; w < TPX / 32; ++w) tot += wcount[w];
    nuniq = tot;
  }
  __syncthreads();
  const int nu = nuniq;
  if (tid < nu) tile_labels[int64_t(tile) * TPX + tid] = uniq[tid];
  if (tid == 0) nslots[tile] = nu;
  if (in) {
    uint8_t sl = kNoSlot;
    if (lab >= 0) {
      int lo = 0, hi = nu - 1;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (uniq[mid] < lab) lo = mid + 1;
        else hi = mid;
      }
      sl = uint8_t(lo);
    }
    slot[i] = sl;
  }
}

__global__ void scatter_partials_kernel(const int32_t* __restrict__ tile_labels,
                                        const int32_t* __restrict__ nslots,
                                        const int32_t* __restrict__ slot_base, int ntiles,
                                        int32_t* __restrict__ partial_comp,
                                        int32_t* __restrict__ partial_idx,
                                        int32_t* __restrict__ comp_ntiles) {
  const int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const int ns = nslots[tile];
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    const int32_t c = tile_labels[int64_t(tile) * TPX + s];
    const int32_t pidx = slot_base[tile] + s;
    partial_comp[pidx] = c;
    partial_idx[pidx] = pidx;
    atomicAdd(comp_ntiles + c, 1);
  }
}

// ------------------------------------------------------- tile reduction

struct TileShared {
  int32_t comp[TPX];
  double coef[TPX];
  uint8_t act[TPX];
  int32_t wcnt[TY];
  int32_t wslot[TY][32];
  double wval[TY][32];
  int32_t last[TPX];
  int32_t nlast;
  int32_t any_active;
  double red[32];
};

// Segmented (by slot) deterministic reduction of v over the tile, write the
// tile's partials, then let the last-arriving CTA of each component reduce
// its partials in plan order and call fin(c, total).
template <class Fin>
__device__ __forceinline__ void tile_reduce(TileShared& sh, const Plan& pl, int tile, int ns,
                                            bool mine, int sl, double v, Fin fin) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  unsigned act = __ballot_sync(0xffffffffu, mine);
  int nent = 0;
  while (act) {
    const int leader = __ffs(act) - 1;
    const int s = __shfl_sync(0xffffffffu, sl, leader);
    const bool in_s = mine && sl == s;
    const double vv = warp_sum(in_s ? v : 0.0);
    if (lane == 0) {
      sh.wslot[w][nent] = s;
      sh.wval[w][nent] = vv;
    }
    ++nent;
    act &= ~__ballot_sync(0xffffffffu, in_s);
  }
  if (lane == 0) sh.wcnt[w] = nent;
  if (tid == 0) sh.nlast = 0;
  __syncthreads();
  const int base = pl.slot_base[tile];
  if (tid < ns && sh.act[tid]) {
    double sum = 0.0;
    for (int ww = 0; ww < TY; ++ww)
      for (int e = 0; e < sh.wcnt[ww]; ++e)
        if (sh.wslot[ww][e] == tid) sum += sh.wval[ww][e];
    pl.partial[base + tid] = sum;
    __threadfence();
    const int32_t c = sh.comp[tid];
    const int32_t n = pl.comp_pstart[c + 1] - pl.comp_pstart[c];
    const int32_t old = atomicAdd(pl.comp_cnt + c, 1);
    if (old == n - 1) sh.last[atomicAdd(&sh.nlast, 1)] = c;
  }
  __syncthreads();
  const int nl = sh.nlast;
  if (nl) __threadfence();
  for (int k = 0; k < nl; ++k) {
    const int32_t c = sh.last[k];
    const int32_t p0 = pl.comp_pstart[c], p1 = pl.comp_pstart[c + 1];
    double sum = 0.0;
    for (int j = p0 + tid; j < p1; j += TPX) sum += __ldcg(pl.partial + pl.comp_plist[j]);
    sum = block_sum(sum, sh.red);
    if (tid == 0) {
      fin(c, sum);
      pl.comp_cnt[c] = 0;
    }
    __syncthreads();
  }
}

// Load the tile's slot table; returns false (uniformly) if nothing is active.
__device__ __forceinline__ bool load_slots(TileShared& sh, const Plan& pl, const FillState& st,
                                           int tile, int ns, int which) {
  const int tid = threadIdx.x;
  if (tid == 0) sh.any_active = 0;
  __syncthreads();
  if (tid < ns) {
    const int32_t c = pl.partial_comp[pl.slot_base[tile] + tid];
    sh.comp[tid] = c;
    const bool a = st.status[c] == ST_ACTIVE;
    sh.act[tid] = a;
    sh.coef[tid] = which == 0 ? st.beta[c] : st.alpha[c];
    if (a) sh.any_active = 1;
  }
  __syncthreads();
  return sh.any_active != 0;
}

// Initial ||b||^2 per component and the state of every component.
__global__ void __launch_bounds__(TPX) init_norm_kernel(Plan pl, FillState st,
                                                        const float* __restrict__ r,
                                                        const uint8_t* __restrict__ slot, int rows,
                                                        int W, double rtol) {
  __shared__ TileShared sh;
  const int tile = blockIdx.x;
  const int ns = pl.nslots[tile];
  if (ns == 0) return;
  const int tid = threadIdx.x;
  if (tid < ns) {
    sh.comp[tid] = pl.partial_comp[pl.slot_base[tile] + tid];
    sh.act[tid] = 1;
  }
  __syncthreads();
  const int tx = tid % TX, ty = tid / TX;
  const int gx = (tile % pl.ntx) * TX + tx, gy = (tile / pl.ntx) * TY + ty;
  int sl = kNoSlot;
  double v = 0.0;
  if (gx < W && gy < rows) {
    const int64_t i = int64_t(gy) * W + gx;
    sl = slot[i];
    if (sl != kNoSlot) {
      const double ri = r[i];
      v = ri * ri;
    }
  }
  tile_reduce(sh, pl, tile, ns, sl != kNoSlot, sl, v, [&](int32_t c, double bb) {
    st.rho[c] = bb;
    const double bn = sqrt(bb);
    st.tol[c] = rtol * bn;
    st.iters[c] = 0;
    st.alpha[c] = 0.0;
    st.beta[c] = 0.0;
    // scipy: bnrm2 == 0 -> x = 0; the first top-of-loop test ||r0|| < rtol ||b||
    if (bb == 0.0 || bn < rtol * bn) {
      st.status[c] = ST_CONVERGED;
    } else if (st.cap[c] <= 0) {
      st.status[c] = ST_CAPPED;
    } else {
      st.status[c] = ST_ACTIVE;
      atomicAdd(st.active, 1);
    }
  });
}

__global__ void init_state_kernel(FillState st, const int32_t* __restrict__ comp_size, int C,
                                  int cg_max_iters) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    st.status[c] = ST_IDLE;
    st.iters[c] = 0;
    const int n = comp_size[c];
    st.cap[c] = n > cg_max_iters ? n : cg_max_iters;
    st.rho[c] = 0.0;
  }
}

// ----------------------------------------------------------------- sweeps

// sweep 1: p = r + beta p ; q = A p ; partial <p, q>  ->  alpha = rho / <p,q>
template <int CONN>
__global__ void __launch_bounds__(TPX) sweep1_kernel(Plan pl, FillState st,
                                                     const float* __restrict__ r,
                                                     float* __restrict__ p, float* __restrict__ q,
                                                     const float* __restrict__ hw,
                                                     const uint8_t* __restrict__ imask,
                                                     const uint8_t* __restrict__ slot, int rows,
                                                     int W) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  __shared__ TileShared sh;
  __shared__ float s_r[TY + 2][TX + 2];
  __shared__ float s_p[TY + 2][TX + 2];
  __shared__ float s_h[TY + 2][TX + 2];
  const int tile = blockIdx.x;
  const int ns = pl.nslots[tile];
  if (ns == 0) return;
  if (!load_slots(sh, pl, st, tile, ns, 0)) return;
  const int tid = threadIdx.x;
  const int x0 = (tile % pl.ntx) * TX, y0 = (tile / pl.ntx) * TY;
  for (int idx = tid; idx < (TY + 2) * (TX + 2); idx += TPX) {
    const int ly = idx / (TX + 2), lx = idx % (TX + 2);
    const int gy = y0 + ly - 1, gx = x0 + lx - 1;
    float rv = 0.f, pv = 0.f, hv = 0.f;
    if (gy >= 0 && gy < rows && gx >= 0 && gx < W) {
      const int64_t j = int64_t(gy) * W + gx;
      rv = r[j];
      pv = p[j];
      hv = hw[j];
    }
    s_r[ly][lx] = rv;
    s_p[ly][lx] = pv;
    s_h[ly][lx] = hv;
  }
  __syncthreads();
  const int tx = tid % TX, ty = tid / TX;
  const int gx = x0 + tx, gy = y0 + ty;
  int sl = kNoSlot;
  bool mine = false;
  double v = 0.0;
  if (gx < W && gy < rows) {
    const int64_t i = int64_t(gy) * W + gx;
    sl = slot[i];
    if (sl != kNoSlot && sh.act[sl]) {
      mine = true;
      const double beta = sh.coef[sl];
      const float pa = float(double(s_r[ty + 1][tx + 1]) + beta * double(s_p[ty + 1][tx + 1]));
      const double ha = s_h[ty + 1][tx + 1];
      const uint8_t m = imask[i];
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
        if ((m >> k) & 1) {
          const int ly = ty + 1 + dv, lx = tx + 1 + du;
          const float pj = float(double(s_r[ly][lx]) + beta * double(s_p[ly][lx]));
          acc += (ha + double(s_h[ly][lx])) * (double(pa) - double(pj));
        }
        if ((m >> (4 + k)) & 1) {
          const int ly = ty + 1 - dv, lx = tx + 1 - du;
          const float pj = float(double(s_r[ly][lx]) + beta * double(s_p[ly][lx]));
          acc += (ha + double(s_h[ly][lx])) * (double(pa) - double(pj));
        }
      }
      const float qa = float(acc);
      p[i] = pa;
      q[i] = qa;
      v = double(pa) * double(qa);
    }
  }
  tile_reduce(sh, pl, tile, ns, mine, sl, v, [&](int32_t c, double pq) {
    if (pq > 0.0) {
      st.alpha[c] = st.rho[c] / pq;
    } else {  // breakdown: p in the null space, only possible once r == 0
      st.alpha[c] = 0.0;
      st.status[c] = ST_CONVERGED;
      atomicSub(st.active, 1);
    }
  });
}

// sweep 2: x += alpha p ; r -= alpha q ; partial <r, r> -> stop test, beta
__global__ void __launch_bounds__(TPX) sweep2_kernel(Plan pl, FillState st, float* __restrict__ x,
                                                     float* __restrict__ r,
                                                     const float* __restrict__ p,
                                                     const float* __restrict__ q,
                                                     const uint8_t* __restrict__ slot, int rows,
                                                     int W) {
  __shared__ TileShared sh;
  const int tile = blockIdx.x;
  const int ns = pl.nslots[tile];
  if (ns == 0) return;
  if (!load_slots(sh, pl, st, tile, ns, 1)) return;
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int gx = (tile % pl.ntx) * TX + tx, gy = (tile / pl.ntx) * TY + ty;
  int sl = kNoSlot;
  bool mine = false;
  double v = 0.0;
  if (gx < W && gy < rows) {
    const int64_t i = int64_t(gy) * W + gx;
    sl = slot[i];
    if (sl != kNoSlot && sh.act[sl]) {
      mine = true;
      const double alpha = sh.coef[sl];
      const double pi = p[i];
      x[i] = float(double(x[i]) + alpha * pi);
      const float rn = float(double(r[i]) - alpha * double(q[i]));
      r[i] = rn;
      v = double(rn) * double(rn);
    }
  }
  tile_reduce(sh, pl, tile, ns, mine, sl, v, [&](int32_t c, double rr) {
    const int it = st.iters[c] + 1;
    st.iters[c] = it;
    // scipy's loop: the test at the top of iteration `it` runs only if it < maxiter
    if (it < st.cap[c] && sqrt(rr) < st.tol[c]) {
      st.status[c] = ST_CONVERGED;
      atomicSub(st.active, 1);
    } else if (it >= st.cap[c]) {
      st.status[c] = ST_CAPPED;
      atomicSub(st.active, 1);
    } else {
      st.beta[c] = rr / st.rho[c];
      st.rho[c] = rr;
    }
  });
}

__global__ void output_kernel(const float* __restrict__ x, const uint8_t* __restrict__ slot,
                              const int32_t* __restrict__ labels, int64_t npix,
                              double* __restrict__ z) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x)
    z[i] = (labels[i] >= 0 && slot[i] != kNoSlot) ? double(x[i]) : 0.0;
}

__global__ void status_out_kernel(const FillState st, int C, int32_t* __restrict__ iters_out,
                                  int32_t* __restrict__ status_out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    iters_out[c] = st.iters[c];
    status_out[c] = st.status[c] == ST_CAPPED ? 1 : 0;
  }
}

// ------------------------------------------------------------ workspace

struct FillWs {
  float *x, *r, *p, *q, *hw;
  uint8_t *imask, *slot;
  int32_t *slot_base, *nslots, *tile_labels, *partial_comp, *partial_idx, *plist, *keys_sorted;
  int32_t *comp_size, *comp_ntiles, *comp_pstart, *comp_cnt, *iters, *cap, *active, *total;
  double *partial, *rho, *alpha, *beta, *tol;
  uint8_t* status;
  void* sort_ws;
  size_t sort_bytes;
  void* scan_ws;
};

static void carve_fill(Carver& c, FillWs& w, int64_t npix, int ntiles, int C) {
  const int64_t P = npix;  // every slot owns >= 1 pixel
  w.x = c.take<float>(npix);
  w.r = c.take<float>(npix);
  w.p = c.take<float>(npix);
  w.q = c.take<float>(npix);
  w.hw = c.take<float>(npix);
  w.imask = c.take<uint8_t>(npix);
  w.slot = c.take<uint8_t>(npix);
  w.slot_base = c.take<int32_t>(ntiles + 1);
  w.nslots = c.take<int32_t>(ntiles + 1);
  w.tile_labels = c.take<int32_t>(int64_t(ntiles) * TPX);
  w.partial_comp = c.take<int32_t>(P);
  w.partial_idx = c.take<int32_t>(P);
  w.plist = c.take<int32_t>(P);
  w.keys_sorted = c.take<int32_t>(P);
  w.partial = c.take<double>(P);
  w.comp_size = c.take<int32_t>(C + 1);
  w.comp_ntiles = c.take<int32_t>(C + 1);
  w.comp_pstart = c.take<int32_t>(C + 1);
  w.comp_cnt = c.take<int32_t>(C + 1);
  w.iters = c.take<int32_t>(C + 1);
  w.cap = c.take<int32_t>(C + 1);
  w.rho = c.take<double>(C + 1);
  w.alpha = c.take<double>(C + 1);
  w.beta = c.take<double>(C + 1);
  w.tol = c.take<double>(C + 1);
  w.status = c.take<uint8_t>(C + 1);
  w.active = c.take<int32_t>(1);
  w.total = c.take<int32_t>(1);
  w.sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, w.sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)P);
  w.sort_ws = c.take<char>(w.sort_bytes);
  const int64_t scan_n = (ntiles + 1) > (C + 1) ? (ntiles + 1) : (C + 1);
  w.scan_ws = c.take<char>(scan_ws_bytes(scan_n));
}

}  // namespace ni

using namespace ni;

extern "C" int ni_fill_workspace_size(int B, int H, int W, int connectivity, int count,
                                      size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  const int64_t npix = int64_t(B) * H * W;
  const int ntiles = div_up(W, TX) * div_up(int64_t(B) * H, TY);
  Sizer s;
  FillWs w;
  carve_fill(s, w, npix, ntiles, count);
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
  const int ntx = div_up(W, TX), nty = div_up(rows, TY);
  const int ntiles = ntx * nty;
  Carver cv(workspace, workspace_bytes);
  FillWs w;
  carve_fill(cv, w, npix, ntiles, count);
  if (!cv.ok() || !workspace) {
    set_error("ni_fill: workspace too small (%zu < %zu)", workspace_bytes, cv.used);
    return NI_ERR_WORKSPACE;
  }
  const int blocks = int(std::min<int64_t>((npix + 255) / 256, int64_t(kSMs) * 16));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_size, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_ntiles, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.comp_cnt, 0, sizeof(int32_t) * (count + 1), s));
  NI_CUDA_TRY(cudaMemsetAsync(w.active, 0, sizeof(int32_t), s));
  if (connectivity == 8)
    prep_kernel<8, 0><<<blocks, 256, 0, s>>>(labels, omega_a, omega_b, gamma, eflags, H, W, npix,
                                             w.hw, w.imask, w.x, w.r, w.p, w.q, w.comp_size);
  else if (model == 0)
    prep_kernel<4, 0><<<blocks, 256, 0, s>>>(labels, omega_a, omega_b, gamma, eflags, H, W, npix,
                                             w.hw, w.imask, w.x, w.r, w.p, w.q, w.comp_size);
  else
    prep_kernel<4, 1><<<blocks, 256, 0, s>>>(labels, omega_a, omega_b, gamma, eflags, H, W, npix,
                                             w.hw, w.imask, w.x, w.r, w.p, w.q, w.comp_size);
  NI_LAUNCH_CHECK();
  // ---- static reduction plan
  tile_slots_kernel<<<ntiles, TPX, 0, s>>>(labels, w.comp_size, rows, W, ntx, w.nslots,
                                          w.tile_labels, w.slot);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(w.nslots, w.slot_base, ntiles, w.total, w.scan_ws, s));
  int32_t P = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&P, w.total, sizeof(P), cudaMemcpyDeviceToHost, s));
  scatter_partials_kernel<<<ntiles, 64, 0, s>>>(w.tile_labels, w.nslots, w.slot_base, ntiles,
                                                w.partial_comp, w.partial_idx, w.comp_ntiles);
  NI_LAUNCH_CHECK();
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  if (P > 0) {
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= count) ++end_bit;
    size_t sb = w.sort_bytes;
    NI_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_ws, sb, w.partial_comp, w.keys_sorted,
                                                w.partial_idx, w.plist, P, 0, end_bit, s));
  }
  NI_TRY(exclusive_scan_i32(w.comp_ntiles, w.comp_pstart, count + 1, nullptr, w.scan_ws, s));
  FillState st{w.rho, w.alpha, w.beta, w.tol, w.iters, w.cap, w.status, w.active};
  Plan pl{ntx, nty, w.slot_base, w.nslots, w.partial_comp, w.comp_pstart, w.plist, w.comp_cnt,
          w.partial};
  if (count > 0) {
    init_state_kernel<<<div_up(count, 256), 256, 0, s>>>(st, w.comp_size, count, cg_max_iters);
    NI_LAUNCH_CHECK();
  }
  init_norm_kernel<<<ntiles, TPX, 0, s>>>(pl, st, w.r, w.slot, rows, W, cg_tol);
  NI_LAUNCH_CHECK();
  // ---- CG iterations: two launches per iteration, convergence polled every
  // `chunk` iterations (finished components cost an early-exit CTA only).
  const int chunk = 16;
  int32_t active = 0;
  NI_CUDA_TRY(cudaMemcpyAsync(&active, w.active, sizeof(active), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  while (active > 0) {
    for (int it = 0; it < chunk; ++it) {
      if (connectivity == 8)
        sweep1_kernel<8><<<ntiles, TPX, 0, s>>>(pl, st, w.r, w.p, w.q, w.hw, w.imask, w.slot, rows,
                                                W);
      else
        sweep1_kernel<4><<<ntiles, TPX, 0, s>>>(pl, st, w.r, w.p, w.q, w.hw, w.imask, w.slot, rows,
                                                W);
      sweep2_kernel<<<ntiles, TPX, 0, s>>>(pl, st, w.x, w.r, w.p, w.q, w.slot, rows, W);
    }
    NI_LAUNCH_CHECK();
    NI_CUDA_TRY(cudaMemcpyAsync(&active, w.active, sizeof(active), cudaMemcpyDeviceToHost, s));
    NI_CUDA_TRY(cudaStreamSynchronize(s));
  }
  output_kernel<<<blocks, 256, 0, s>>>(w.x, w.slot, labels, npix, z_out);
  NI_LAUNCH_CHECK();
  if (count > 0) {
    status_out_kernel<<<div_up(count, 256), 256, 0, s>>>(st, count, comp_iters, comp_status);
    NI_LAUNCH_CHECK();
  }
  return NI_OK;
}

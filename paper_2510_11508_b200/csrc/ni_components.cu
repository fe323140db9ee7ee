// K0 (NormalMap.create) and K1 (form_components) on the pixel grid.
//
// K0 reproduces geometry.py:123-145 bit for bit: float64 norm
// sqrt((x0*x0 + x1*x1) + x2*x2) with IEEE products/sums (no FMA), IEEE
// division.  K1 reproduces graph.py:89-98 + 141-165: the kept-edge predicate
// is the float64 dot ((a0*b0 + a1*b1) + a2*b2) >= d*, where the host passes
// d* = the smallest float64 whose numpy arccos is < theta_c, so the kept set
// is bit-identical to arccos(clip(dot)) < theta_c.  Components are found by a
// lock-free union-find (roots hooked under the smaller id with atomicMin, so
// every root is its component's smallest pixel id) and ranked by an
// exclusive scan of the root flags, which is exactly the canonical labelling
// of graph.py:133-138 (rank of the smallest row-major id).
#include "ni_common.cuh"

namespace ni {

// ------------------------------------------------------------------ K0

template <typename T>
__global__ void __launch_bounds__(256) normalize_kernel(const T* __restrict__ in,
                                                        const uint8_t* __restrict__ mask,
                                                        int64_t npix, double* __restrict__ n_out,
                                                        uint8_t* __restrict__ valid_out,
                                                        ni_stats* __restrict__ st) {
  long long nvalid = 0, nnonfin = 0, nnonunit = 0;
  unsigned long long maxdev = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool m = mask ? mask[i] != 0 : true;
    double o0 = 0.0, o1 = 0.0, o2 = 0.0;
    if (m) {
      const double x0 = double(in[3 * i + 0]);
      const double x1 = double(in[3 * i + 1]);
      const double x2 = double(in[3 * i + 2]);
      ++nvalid;
      if (!(isfinite(x0) && isfinite(x1) && isfinite(x2))) {
        ++nnonfin;
      } else {
        const double nrm = __dsqrt_rn(add_rn(add_rn(mul_rn(x0, x0), mul_rn(x1, x1)), mul_rn(x2, x2)));
        const double dev = fabs(__dadd_rn(nrm, -1.0));
        if (dev > 1e-4) {
          ++nnonunit;
          unsigned long long b = __double_as_longlong(dev);
          maxdev = b > maxdev ? b : maxdev;
        }
        o0 = __ddiv_rn(x0, nrm);
        o1 = __ddiv_rn(x1, nrm);
        o2 = __ddiv_rn(x2, nrm);
      }
    }
    valid_out[i] = m ? 1 : 0;
    n_out[i] = o0;
    n_out[npix + i] = o1;
    n_out[2 * npix + i] = o2;
  }
  // one atomic per warp per counter (integer: order-independent)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
    nnonfin += __shfl_xor_sync(0xffffffffu, nnonfin, o);
    nnonunit += __shfl_xor_sync(0xffffffffu, nnonunit, o);
    unsigned long long t = __shfl_xor_sync(0xffffffffu, maxdev, o);
    maxdev = t > maxdev ? t : maxdev;
  }
  if ((threadIdx.x & 31) == 0) {
    if (nvalid) atomicAdd((unsigned long long*)&st->valid_pixels, (unsigned long long)nvalid);
    if (nnonfin) atomicAdd((unsigned long long*)&st->nonfinite, (unsigned long long)nnonfin);
    if (nnonunit) atomicAdd((unsigned long long*)&st->nonunit, (unsigned long long)nnonunit);
    if (maxdev) atomicMax(&st->max_dev, maxdev);
  }
}

// ------------------------------------------------------------------ K1

// Tiled K1: union-find inside 32 x 32 tiles in shared memory (local ids are
// row-major within the tile, so the smaller local id is the smaller pixel
// id), then one global union per kept edge that leaves its tile.
constexpr int UT = 32;  // tile edge

__device__ __forceinline__ bool kept_edge(const double* __restrict__ n, int64_t npix, int64_t i,
                                          int64_t j, double cutoff, int theta_none) {
  if (theta_none) return false;
  const double d = add_rn(add_rn(mul_rn(n[i], n[j]), mul_rn(n[npix + i], n[npix + j])),
                          mul_rn(n[2 * npix + i], n[2 * npix + j]));
  return d >= cutoff;
}

__device__ __forceinline__ int sm_find(volatile int* p, int x) {
  int q = p[x];
  while (q != x) {
    const int gq = p[q];
    if (gq != q) p[x] = gq;
    x = gq;
    q = p[x];
  }
  return x;
}

__device__ __forceinline__ void sm_union(int* p, int a, int b) {
  volatile int* vp = p;
  while (true) {
    a = sm_find(vp, a);
    b = sm_find(vp, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(p + a, b);
    if (old == a) return;
    a = old;
  }
}

// One 32 x 32 tile per CTA (warp w owns rows w, w+8, w+16, w+24; lane =
// column).  (1) The kept-edge bits of every in-tile forward edge.  (2) Row
// runs: pixels joined by kept right edges share the run's first pixel as
// parent, found with one warp ballot per row (no atomics).  (3) Union-find in
// shared memory over the remaining edges, skipping every edge another pair of
// kept edges already implies (a down edge whose left neighbour's down edge
// joins the same two runs; a diagonal closed by a right + down pair): a
// uniform region then needs one union per row instead of four per pixel.
// Roots stay the smallest local id, i.e. the smallest pixel id.
template <int CONN>
__global__ void __launch_bounds__(256) uf_tile_kernel(const double* __restrict__ n,
                                                      const uint8_t* __restrict__ valid, int H,
                                                      int W, int64_t rows, int tiles_x,
                                                      double cutoff, int theta_none,
                                                      int32_t* __restrict__ parent,
                                                      ni_stats* __restrict__ st) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  // edge bits: 0 right, 1 down, 2 down-left, 3 down-right (in-tile, kept)
  constexpr uint8_t RT = 1, DN = 2, DL = 4, DR = 8;
  __shared__ int p[UT * UT];
  __shared__ uint8_t kb[UT * UT];
  __shared__ double sn[3][UT * UT];  // the tile's normals: in-tile edges read only these
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int x0 = tx * UT;
  const int64_t y0 = int64_t(ty) * UT;
  const int64_t npix = rows * W;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int l = threadIdx.x; l < UT * UT; l += blockDim.x) {
    const int x = x0 + (l % UT);
    const int64_t y = y0 + l / UT;
    const bool in = x < W && y < rows;
    const int64_t gi = y * W + x;
    p[l] = (in && valid[gi]) ? l : -1;
    if (in) {
      sn[0][l] = n[gi];
      sn[1][l] = n[npix + gi];
      sn[2][l] = n[2 * npix + gi];
    }
  }
  __syncthreads();
  long long nedges = 0;
  // (1) kept bits
#pragma unroll
  for (int q = 0; q < UT / 8; ++q) {
    const int ly = wid + 8 * q, lx = lane, l = ly * UT + lx;
    uint8_t bits = 0;
    if (p[l] >= 0) {
      const int x = x0 + lx;
      const int64_t y = y0 + ly;
      const int64_t i = y * W + x;
      const int vloc = int(uint32_t(y) % uint32_t(H));
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
        if (!fwd_inside(x, vloc, du, dv, W, H)) continue;
        const int64_t j = i + int64_t(dv) * W + du;
        const int jx = lx + du, jy = ly + dv;
        const bool inside = jx >= 0 && jx < UT && jy < UT;
        if (inside ? p[jy * UT + jx] < 0 : !valid[j]) continue;
        ++nedges;
        if (!inside || theta_none) continue;  // crosses the tile: the border pass
        const int lj = jy * UT + jx;
        if (add_rn(add_rn(mul_rn(sn[0][l], sn[0][lj]), mul_rn(sn[1][l], sn[1][lj])),
                   mul_rn(sn[2][l], sn[2][lj])) >= cutoff) {  // = kept_edge(n, npix, i, j, ...)
          const uint8_t b = du == 1 && dv == 0 ? RT : (du == 0 ? DN : (du < 0 ? DL : DR));
          bits |= b;
        }
      }
    }
    kb[l] = bits;
  }
  __syncwarp();
  // (2) row runs: a pixel starts a run unless its left neighbour's right edge is kept
#pragma unroll
  for (int q = 0; q < UT / 8; ++q) {
    const int ly = wid + 8 * q, l = ly * UT + lane;
    const uint8_t left = __shfl_up_sync(0xffffffffu, kb[l], 1);
    const bool start = lane == 0 || !(left & RT);
    const unsigned starts = __ballot_sync(0xffffffffu, start);
    const unsigned upto = starts & (0xffffffffu >> (31 - lane));
    if (p[l] >= 0) p[l] = ly * UT + (31 - __clz(upto));
  }
  __syncthreads();
  // (3) the remaining (non-implied) edges
#pragma unroll
  for (int q = 0; q < UT / 8; ++q) {
    const int ly = wid + 8 * q, l = ly * UT + lane;
    const uint8_t b = kb[l];
    if (ly == UT - 1 || !(b & (DN | DL | DR))) continue;
    const uint8_t bl = lane > 0 ? kb[l - 1] : 0;   // left neighbour
    const uint8_t br = lane < UT - 1 ? kb[l + 1] : 0;  // right neighbour
    const uint8_t dnb = kb[l + UT];                       // pixel below
    const uint8_t dlb = lane > 0 ? kb[l + UT - 1] : 0;    // below-left
    if (b & DN) {
      // implied by the left neighbour's down edge when both row pairs are runs
      const bool implied = (bl & RT) && (bl & DN) && (dlb & RT);
      if (!implied) sm_union(p, l, l + UT);
    }
    if (b & DR) {  // (x, y) -> (x + 1, y + 1)
      const bool implied = ((b & RT) && (br & DN)) || ((b & DN) && (dnb & RT));
      if (!implied) sm_union(p, l, l + UT + 1);
    }
    if (b & DL) {  // (x, y) -> (x - 1, y + 1)
      const bool implied = ((bl & RT) && (bl & DN)) || ((b & DN) && (dlb & RT));
      if (!implied) sm_union(p, l, l + UT - 1);
    }
  }
  __syncthreads();
  for (int l = threadIdx.x; l < UT * UT; l += blockDim.x) {
    const int x = x0 + (l % UT);
    const int64_t y = y0 + l / UT;
    if (x >= W || y >= rows) continue;
    const int64_t gi = y * W + x;
    if (p[l] < 0) {
      parent[gi] = -1;  // invalid pixel
      continue;
    }
    const int r = sm_find(p, l);
    parent[gi] = int32_t((y0 + r / UT) * W + x0 + (r % UT));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nedges += __shfl_xor_sync(0xffffffffu, nedges, o);
  if ((threadIdx.x & 31) == 0 && nedges)
    atomicAdd((unsigned long long*)&st->edges, (unsigned long long)nedges);
}

// kept edges that leave their tile, unioned in global memory.  Only pixels
// on a tile's left / right column or bottom row have such edges (forward
// offsets point right or down): the grid enumerates those 3 * UT - 2
// positions per tile instead of every pixel.
constexpr int UT_BORDER = 3 * UT - 2;

template <int CONN>
__global__ void __launch_bounds__(256) uf_border_kernel(const double* __restrict__ n,
                                                        const uint8_t* __restrict__ valid, int H,
                                                        int W, int64_t rows, int tiles_x,
                                                        int64_t nslots, double cutoff,
                                                        int theta_none, int32_t* parent) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  const int64_t npix = rows * W;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nslots;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tile = t / UT_BORDER;
    const int pos = int(t - tile * UT_BORDER);
    int lx, ly;
    if (pos < UT) {  // left column
      lx = 0;
      ly = pos;
    } else if (pos < 2 * UT) {  // right column
      lx = UT - 1;
      ly = pos - UT;
    } else {  // bottom row between the corners
      lx = pos - 2 * UT + 1;
      ly = UT - 1;
    }
    const int x = int(tile % tiles_x) * UT + lx;
    const int64_t y = (tile / tiles_x) * UT + ly;
    if (x >= W || y >= rows) continue;
    const int64_t i = y * W + x;
    if (!valid[i]) continue;
    const int vloc = int(y % H);
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
      const int jx = lx + du, jy = ly + dv;
      if (jx >= 0 && jx < UT && jy < UT) continue;  // inside: done by the tile pass
      if (!fwd_inside(x, vloc, du, dv, W, H)) continue;
      const int64_t j = i + int64_t(dv) * W + du;
      if (!valid[j]) continue;
      if (kept_edge(n, npix, i, j, cutoff, theta_none)) uf_union(parent, int32_t(i), int32_t(j));
    }
  }
}

__global__ void uf_flatten_kernel(int32_t* parent, int64_t npix, int32_t* __restrict__ root_flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    int32_t p = parent[i];
    if (p < 0) {
      root_flag[i] = 0;
      continue;
    }
    int32_t r = uf_find(parent, int32_t(i));
    parent[i] = r;
    root_flag[i] = (r == int32_t(i)) ? 1 : 0;
  }
}

__global__ void relabel_kernel(const int32_t* __restrict__ parent, const int32_t* __restrict__ rank,
                               int64_t npix, int32_t* __restrict__ labels) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    int32_t p = parent[i];
    labels[i] = p < 0 ? -1 : rank[p];
  }
}

__global__ void map_first_kernel(const int32_t* __restrict__ rank, const int32_t* __restrict__ total,
                                 int B, int64_t per_map, int32_t* __restrict__ map_first,
                                 int32_t* __restrict__ count) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < B) map_first[m] = rank[int64_t(m) * per_map];
  if (m == B) {
    map_first[B] = total[0];
    count[0] = total[0];
  }
}

static int grid_blocks(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = int64_t(kSMs) * 16;
  return int(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace ni

using namespace ni;

extern "C" int ni_normalize(const void* normals, int dtype, const uint8_t* mask, int B, int H, int W,
                            double* n_out, uint8_t* valid_out, ni_stats* stats, ni_stream_t stream) {
  NI_CHECK_ARG(B >= 1 && H >= 1 && W >= 1, "grid dimensions must be positive");
  NI_CHECK_ARG(int64_t(B) * H * W < (int64_t(1) << 31) - 1, "grid larger than 2^31-1 pixels");
  NI_CHECK_ARG(dtype == 0 || dtype == 1, "dtype must be 0 (float32) or 1 (float64)");
  NI_CHECK_ARG(normals && n_out && valid_out && stats, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  NI_CUDA_TRY(cudaMemsetAsync(stats, 0, sizeof(ni_stats), s));
  const int blocks = grid_blocks(npix);
  if (dtype == 0)
    NI_COUNT_LAUNCH(), normalize_kernel<float><<<blocks, 256, 0, s>>>((const float*)normals, mask, npix, n_out,
                                                  valid_out, stats);
  else
    NI_COUNT_LAUNCH(), normalize_kernel<double><<<blocks, 256, 0, s>>>((const double*)normals, mask, npix, n_out,
                                                   valid_out, stats);
  NI_LAUNCH_CHECK();
  ni_stats h;
  NI_CUDA_TRY(cudaMemcpyAsync(&h, stats, sizeof(h), cudaMemcpyDeviceToHost, s));
  NI_CUDA_TRY(cudaStreamSynchronize(s));
  if (h.nonfinite) {
    set_error("valid normals must be finite (%lld non-finite)", h.nonfinite);
    return NI_ERR_NONFINITE;
  }
  if (h.nonunit) {
    double worst;
    memcpy(&worst, &h.max_dev, sizeof(worst));
    set_error("%lld valid normals deviate from unit norm by up to %.3g (tolerance 0.0001)", h.nonunit,
              worst);
    return NI_ERR_NONUNIT_NORMAL;
  }
  if (h.valid_pixels == 0) {
    set_error("normal map has no valid pixel");
    return NI_ERR_EMPTY_MASK;
  }
  return NI_OK;
}

extern "C" int ni_components_workspace_size(int B, int H, int W, size_t* bytes) {
  NI_CHECK_ARG(bytes, "null pointer");
  const int64_t npix = int64_t(B) * H * W;
  Sizer z;
  z.take<int32_t>(npix);  // parent
  z.take<int32_t>(npix);  // root flags
  z.take<int32_t>(npix);  // rank
  z.take<int32_t>(1);     // total
  z.take<char>(scan_ws_bytes(npix));
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_components(const double* n, const uint8_t* valid, int B, int H, int W,
                             int connectivity, double dot_cutoff, int theta_none, int32_t* labels_out,
                             int32_t* count_out, int32_t* map_first_out, ni_stats* stats,
                             void* workspace, size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(B >= 1 && H >= 1 && W >= 1, "grid dimensions must be positive");
  NI_CHECK_ARG(n && valid && labels_out && count_out && map_first_out && stats, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  Carver c(workspace, workspace_bytes);
  int32_t* parent = c.take<int32_t>(npix);
  int32_t* flags = c.take<int32_t>(npix);
  int32_t* rank = c.take<int32_t>(npix);
  int32_t* total = c.take<int32_t>(1);
  void* scan_ws = c.take<char>(scan_ws_bytes(npix));
  if (!c.ok() || !workspace) {
    set_error("ni_components: workspace too small (%zu < %zu)", workspace_bytes, c.used);
    return NI_ERR_WORKSPACE;
  }
  NI_CUDA_TRY(cudaMemsetAsync(&stats->edges, 0, sizeof(long long), s));
  const int blocks = grid_blocks(npix);
  const int64_t rows = int64_t(B) * H;
  const int tiles_x = div_up(W, UT);
  const int64_t tiles = int64_t(tiles_x) * div_up(rows, UT);
  NI_CHECK_ARG(tiles < (int64_t(1) << 31), "grid too large");
  if (connectivity == 8) {
    NI_COUNT_LAUNCH(), uf_tile_kernel<8><<<int(tiles), 256, 0, s>>>(
                           n, valid, H, W, rows, tiles_x, dot_cutoff, theta_none, parent, stats);
    NI_COUNT_LAUNCH(), uf_border_kernel<8><<<grid_blocks(tiles * UT_BORDER), 256, 0, s>>>(
                           n, valid, H, W, rows, tiles_x, tiles * UT_BORDER, dot_cutoff, theta_none,
                           parent);
  } else {
    NI_COUNT_LAUNCH(), uf_tile_kernel<4><<<int(tiles), 256, 0, s>>>(
                           n, valid, H, W, rows, tiles_x, dot_cutoff, theta_none, parent, stats);
    NI_COUNT_LAUNCH(), uf_border_kernel<4><<<grid_blocks(tiles * UT_BORDER), 256, 0, s>>>(
                           n, valid, H, W, rows, tiles_x, tiles * UT_BORDER, dot_cutoff, theta_none,
                           parent);
  }
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), uf_flatten_kernel<<<blocks, 256, 0, s>>>(parent, npix, flags);
  NI_LAUNCH_CHECK();
  NI_TRY(exclusive_scan_i32(flags, rank, npix, total, scan_ws, s));
  NI_COUNT_LAUNCH(), relabel_kernel<<<blocks, 256, 0, s>>>(parent, rank, npix, labels_out);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), map_first_kernel<<<div_up(B + 1, 128), 128, 0, s>>>(rank, total, B, int64_t(H) * W, map_first_out,
                                                      count_out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

// Pixel-edge weights and energies for the weighted fill passes:
//
//  * ni_edge_weights  continuity.py:292-331 / solver.py:253-278 on every
//                     forward pixel edge: the weights of the refill pass
//                     (solver.py:213-216, 237-238) and of each iteration of
//                     the pixel-level baseline (pipeline.py:261-285)
//  * ni_pair_energy   E = sum_e W_a res_a^2 + W_b res_b^2 of the pixel pair
//                     system at x (pipeline.py:336-337), one value per map
//
// Weights are stored as forward-edge planes w[k * npix + a] (edge a -> a +
// offset_k), like the continuity coefficients.
#include "ni_common.cuh"
#include "ni_edges.cuh"

namespace ni {

template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) edge_weights_kernel(
    const double* __restrict__ z, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ gamma,
    const uint8_t* __restrict__ eflags, int H, int W, int64_t npix, WeightArgs wp,
    double* __restrict__ w_a, double* __restrict__ w_b) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npix;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t ef = eflags[i];
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      double wa = 0.0, wb = 0.0;
      if ((ef >> k) & 1)
        edge_weights_at<CONN, MODEL>(z, nullptr, nullptr, omega_a, omega_b, gamma, eflags, H, W, npix, i, k, wp, wa,
                                     wb);
      w_a[k * npix + i] = wa;
      w_b[k * npix + i] = wb;
    }
  }
}

// Per-map energy of the pixel pair system, in a fixed order: CHUNKS blocks
// per map each sum a contiguous pixel range (thread-strided partials + block
// tree), then one thread per map adds its chunks in order.
constexpr int kEnergyChunks = 64;

template <int CONN, int MODEL>
__global__ void __launch_bounds__(256) pair_energy_kernel(
    const double* __restrict__ x, const double* __restrict__ omega_a,
    const double* __restrict__ omega_b, const double* __restrict__ w_a,
    const double* __restrict__ w_b, const uint8_t* __restrict__ eflags, int W, int64_t per_map,
    int64_t npix, double* __restrict__ partial) {
  constexpr int KF = CONN == 8 ? 4 : 2;
  __shared__ double red[32];
  const int m = blockIdx.x / kEnergyChunks, ch = blockIdx.x % kEnergyChunks;
  const int64_t len = (per_map + kEnergyChunks - 1) / kEnergyChunks;
  const int64_t p0 = int64_t(m) * per_map + ch * len;
  const int64_t p1 = min(p0 + len, int64_t(m + 1) * per_map);
  double e = 0.0;
  for (int64_t i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
    const uint8_t ef = eflags[i];
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      if (!((ef >> k) & 1)) continue;
      const int64_t b = i + int64_t(fwd_dv(CONN, k)) * W + fwd_du(CONN, k);
      const double oa = omega_a[k * npix + i];
      const double ob = MODEL == 0 ? -oa : omega_b[k * npix + i];
      const double ra = x[i] - x[b] - oa, rb = x[b] - x[i] - ob;
      e += ra * (w_a[k * npix + i] * ra) + rb * (w_b[k * npix + i] * rb);
    }
  }
  e = block_sum(e, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = e;
}

__global__ void energy_sum_kernel(const double* __restrict__ partial, int B,
                                  double* __restrict__ out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= B) return;
  double e = 0.0;
  for (int c = 0; c < kEnergyChunks; ++c) e += partial[m * kEnergyChunks + c];
  out[m] = e;
}

static int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = int64_t(kSMs) * 16;
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace ni

using namespace ni;

extern "C" int ni_edge_weights(const double* z, const double* omega_a, const double* omega_b,
                               const double* gamma, const uint8_t* eflags, int B, int H, int W,
                               int connectivity, int model, int wmode, int mode, double k,
                               double outlier_low, double outlier_high, double* w_a, double* w_b,
                               ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(model == 0 || (model == 1 && connectivity == 4), "bad model/connectivity");
  NI_CHECK_ARG(wmode >= 0 && wmode <= 2 && mode >= 0 && mode <= 2, "bad weight mode");
  NI_CHECK_ARG(z && omega_a && gamma && eflags && w_a && w_b, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npix = int64_t(B) * H * W;
  WeightArgs wp;
  wp.wmode = wmode;
  wp.mode = mode;
  wp.k = k;
  wp.lt = log10(outlier_low);
  wp.ut = log10(outlier_high);
  wp.hi = outlier_high;
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), edge_weights_kernel<8, 0><<<grid_for(npix), 256, 0, s>>>(
                           z, omega_a, omega_b, gamma, eflags, H, W, npix, wp, w_a, w_b);
  else if (model == 0)
    NI_COUNT_LAUNCH(), edge_weights_kernel<4, 0><<<grid_for(npix), 256, 0, s>>>(
                           z, omega_a, omega_b, gamma, eflags, H, W, npix, wp, w_a, w_b);
  else
    NI_COUNT_LAUNCH(), edge_weights_kernel<4, 1><<<grid_for(npix), 256, 0, s>>>(
                           z, omega_a, omega_b, gamma, eflags, H, W, npix, wp, w_a, w_b);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

extern "C" int ni_pair_energy_workspace_size(int B, size_t* bytes) {
  NI_CHECK_ARG(bytes && B >= 1, "bad argument");
  Sizer z;
  z.take<double>(int64_t(B) * kEnergyChunks);
  *bytes = z.used;
  return NI_OK;
}

extern "C" int ni_pair_energy(const double* x, const double* omega_a, const double* omega_b,
                              const double* w_a, const double* w_b, const uint8_t* eflags, int B,
                              int H, int W, int connectivity, int model, double* energy_out,
                              void* workspace, size_t workspace_bytes, ni_stream_t stream) {
  NI_CHECK_ARG(connectivity == 4 || connectivity == 8, "connectivity must be 4 or 8");
  NI_CHECK_ARG(model == 0 || (model == 1 && connectivity == 4), "bad model/connectivity");
  cudaStream_t s = (cudaStream_t)stream;
  Carver c(workspace, workspace_bytes);
  double* partial = c.take<double>(int64_t(B) * kEnergyChunks);
  if (!c.ok() || !workspace) {
    set_error("ni_pair_energy: workspace too small");
    return NI_ERR_WORKSPACE;
  }
  const int64_t per_map = int64_t(H) * W, npix = per_map * B;
  const int blocks = B * kEnergyChunks;
  if (connectivity == 8)
    NI_COUNT_LAUNCH(), pair_energy_kernel<8, 0><<<blocks, 256, 0, s>>>(
                           x, omega_a, omega_b, w_a, w_b, eflags, W, per_map, npix, partial);
  else if (model == 0)
    NI_COUNT_LAUNCH(), pair_energy_kernel<4, 0><<<blocks, 256, 0, s>>>(
                           x, omega_a, omega_b, w_a, w_b, eflags, W, per_map, npix, partial);
  else
    NI_COUNT_LAUNCH(), pair_energy_kernel<4, 1><<<blocks, 256, 0, s>>>(
                           x, omega_a, omega_b, w_a, w_b, eflags, W, per_map, npix, partial);
  NI_LAUNCH_CHECK();
  NI_COUNT_LAUNCH(), energy_sum_kernel<<<div_up(B, 128), 128, 0, s>>>(partial, B, energy_out);
  NI_LAUNCH_CHECK();
  return NI_OK;
}

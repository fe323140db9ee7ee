// Directed edge weights shared by the relative-scale step (inter edges), the
// reweighted refill pass and the pixel-level baseline (all pixel edges).
#pragma once

#include "ni_common.cuh"

namespace ni {

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// What a weight evaluation includes:
//   EW_UNIFORM   valid                                  (solver.py:269-271, t < alignment_iters)
//   EW_BILATERAL valid * gamma^2 * bilateral(z)         (edge_weights, continuity.py:292-331;
//                                                        the refill pass, solver.py:213-216)
//   EW_FULL      EW_BILATERAL * outlier weight of chi   (solver.py:272-278)
enum : int { EW_UNIFORM = 0, EW_BILATERAL = 1, EW_FULL = 2 };

struct WeightArgs {
  int wmode;   // EW_*
  int mode;    // outlier reweighting: 0 off, 1 soft, 2 hard (continuity.py:140-158)
  double k;    // bilateral sharpness
  double lt;   // log10(outlier_low)
  double ut;   // log10(outlier_high)
  double hi;   // outlier_high
};

// Weights (W_a, W_b) of the two directed rows of forward edge k at pixel a
// (b = a + offset_k), at log-depth state z.  Invalid edges get 0.
// Log-depth at pixel x: z[x], plus the pixel's component shift when the
// caller defers the scale application (zs != nullptr: z_eff = z + zs[label]).
// (zs is not __restrict__: the fused scale loop advances the shifts inside the
// kernel that reads them, so they must not take the non-coherent load path)
__device__ __forceinline__ double z_at(const double* __restrict__ z, const double* zs,
                                       const int32_t* __restrict__ labels, int64_t x) {
  return zs ? z[x] + zs[labels[x]] : z[x];
}

template <int CONN, int MODEL>
__device__ __forceinline__ void edge_weights_at(const double* __restrict__ z,
                                                const double* zs,
                                                const int32_t* __restrict__ zlab,
                                                const double* __restrict__ omega_a,
                                                const double* __restrict__ omega_b,
                                                const double* __restrict__ gamma,
                                                const uint8_t* __restrict__ eflags, int H, int W,
                                                int64_t npix, int64_t a, int k,
                                                const WeightArgs& p, double& wa, double& wb) {
  wa = 0.0;
  wb = 0.0;
  if (!((eflags[a] >> (4 + k)) & 1)) return;  // degenerate coefficient
  if (p.wmode == EW_UNIFORM) {
    wa = wb = 1.0;
    return;
  }
  const int du = fwd_du(CONN, k), dv = fwd_dv(CONN, k);
  const int64_t b = a + int64_t(dv) * W + du;
  const double za = z_at(z, zs, zlab, a), zb = z_at(z, zs, zlab, b);
  // opposite of b through a: a - off (continuity.py:196-207, 276)
  const int ua = int(a % W), va = int((a / W) % H);
  const int uo = ua - du, vo = va - dv;
  bool has_a = false;
  double zoa = 0.0;
  if (uo >= 0 && uo < W && vo >= 0) {
    const int64_t o = a - int64_t(dv) * W - du;
    if ((eflags[o] >> k) & 1) {  // edge o -> a exists: o valid, same map
      has_a = true;
      zoa = z_at(z, zs, zlab, o);
    }
  }
  const bool has_b = (eflags[b] >> k) & 1;  // b + off exists
  const double zob = has_b ? z_at(z, zs, zlab, b + int64_t(dv) * W + du) : 0.0;
  const double ga = gamma[a], gb = gamma[b];
  const double g2a = ga * ga, g2b = gb * gb;
  double bil_a = 0.5, bil_b = 0.5;
  if (has_a) {
    const double dp = zoa - za, dq = zb - za;
    bil_a = sigmoid(p.k * (g2a * (dp * dp - dq * dq)));
  }
  if (has_b) {
    const double dp = zob - zb, dq = za - zb;
    bil_b = sigmoid(p.k * (g2b * (dp * dp - dq * dq)));
  }
  wa = g2a * bil_a;
  wb = g2b * bil_b;
  if (p.wmode != EW_FULL) return;
  // outlier weights on chi (continuity.py:140-158)
  const double oa = omega_a[k * npix + a];
  const double ob = MODEL == 0 ? -oa : omega_b[k * npix + a];
  const double chia = za - zb - oa, chib = zb - za - ob;
  if (p.mode == 1) {
    const double ca = fabs(chia) > 1e-300 ? fabs(chia) : 1e-300;
    const double cb = fabs(chib) > 1e-300 ? fabs(chib) : 1e-300;
    const double sc = 4.0 / (p.lt - p.ut);
    wa *= sigmoid(sc * (2.0 * log10(ca) - (p.lt + p.ut)));
    wb *= sigmoid(sc * (2.0 * log10(cb) - (p.lt + p.ut)));
  } else if (p.mode == 2) {
    if (fabs(chia) >= p.hi) wa = 0.0;
    if (fabs(chib) >= p.hi) wb = 0.0;
  }
}

}  // namespace ni

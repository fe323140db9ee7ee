"""Shared parity criteria (north star, BASELINE.json):

* labels: bit-exact (both sides are canonical: rank of the smallest pixel id);
* depth: exp(log_depth) after the reference's own median gauge,
  mean |d_a - d_b| <= 1e-3 px + 1e-4 * mean |d_b| (allclose-style; SURVEY.md
  Appendix B).  ``px_scale`` converts gauge-fixed depth (median 1) to pixels.
"""

import numpy as np

RTOL = 1e-4
ATOL_PX = 1e-3


def depth_error(log_a, log_b, mask, px_scale=1.0):
    da = np.exp(np.asarray(log_a, np.float64)[mask])
    db = np.exp(np.asarray(log_b, np.float64)[mask])
    mean_abs = float(np.mean(np.abs(da - db)))
    bound = ATOL_PX / px_scale + RTOL * float(np.mean(np.abs(db)))
    return mean_abs, bound


def assert_depth_close(log_a, log_b, mask, px_scale=1.0, what="depth"):
    err, bound = depth_error(log_a, log_b, mask, px_scale)
    assert err <= bound, f"{what}: mean |d| error {err:.3e} > bound {bound:.3e}"


def px_scale_of(intr, mask, log_depth_true=None):
    """Depth units per pixel: the focal length (fx) for the pinhole
    stand-in, i.e. at depth f one pixel spans one depth unit."""
    return float(intr[0])

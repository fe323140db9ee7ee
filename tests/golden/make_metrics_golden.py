"""Golden fixtures for the evaluation metrics (metrics.py:44-113), made by the
REAL reference in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_metrics_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from normint import metrics as M  # noqa: E402
from normint.graph import Partition  # noqa: E402


def case(seed, h, w, ncomp, bad_frac):
    rng = np.random.default_rng(seed)
    gt = 1500.0 + 200.0 * rng.random((h, w))
    comp = rng.integers(0, ncomp, size=(h, w))
    comp_scale = np.exp(rng.normal(0.0, 0.3, ncomp))
    pred = gt * comp_scale[comp] * (1.0 + rng.normal(0.0, 0.01, (h, w))) / 1234.5
    mask = rng.random((h, w)) > 0.1
    bad = rng.random((h, w)) < bad_frac
    pred = np.where(bad & (rng.random((h, w)) < 0.5), np.nan, pred)
    pred = np.where(bad & (rng.random((h, w)) < 0.5), -1.0, pred)
    labels = np.where(mask, comp, -1).ravel()
    # canonical-ish labels are not required by the metric; keep them compact
    p = Partition(labels.astype(np.int64), ncomp)
    rep = M.evaluate(pred, gt, mask)
    mtm = M.min_theoretical_made(pred, gt, p, mask)
    ok = np.isfinite(pred) & (pred > 0) & mask
    l1 = M.l1_optimal_scale(pred[ok][:500], gt[ok][:500])
    return dict(pred=pred, gt=gt, mask=mask, labels=labels.astype(np.int32), ncomp=ncomp,
                made=rep.made, relative_error=rep.relative_error, aligned_scale=rep.aligned_scale,
                valid_pixel_count=rep.valid_pixel_count, min_theoretical_made=mtm, l1_scale=l1)


if __name__ == "__main__":
    for name, args in {"metrics_a": (1, 48, 40, 7, 0.05), "metrics_b": (2, 33, 57, 20, 0.2),
                       "metrics_c": (3, 64, 64, 1, 0.0)}.items():
        d = case(*args)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, d["made"], d["min_theoretical_made"], d["valid_pixel_count"])

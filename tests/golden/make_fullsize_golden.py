"""Compact full-size fixtures from the REAL reference ``normint`` on the
BASELINE configurations (C1, C2, C3, C4 with merging every 5, and the C5
maps 0 / 21 / 42 / 63 the bench batch contains).

Run in the build container only (the reference does not exist on the GPU
box; the inputs are regenerated there from the same seeds by
``paper_2510_11508_b200.scenes``, and a SHA-256 of the float32 normals pins
that both sides saw the same bits):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_golden.py [C1 C2 ...]

Stored per case (``tests/golden/full/<case>.npz``):
* ``labels0`` / ``labels`` -- partition0 and the final partition (int32,
  compressed: one label plane of 16.8 M px is a few hundred KB);
* ``iterations``, ``energies``, ``records`` (without wall_ms), ``warnings``;
* ``scales`` -- the per-component scale of every partition0 component,
  final log-depth - filled log-depth (constant on a component; the gauge
  shift is part of it, identically on both sides);
* ``sample_idx`` / ``log_depth_s`` / ``filled_s`` -- a 1-in-``STRIDE`` sample
  of the valid pixels' final and filled log-depth;
* ``mean_depth`` -- mean exp(log_depth) over the valid pixels;
* ``scale_cg_capped`` -- does any outer iteration's scale CG hit its cap
  (``iteration t: cg hit iteration cap``, pipeline.py:179-180)?  False on
  every BASELINE config: the oracle's range projection of the scale RHS
  (oracle.project_range) is then a no-op on them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2510_11508_b200 import scenes  # noqa: E402

import normint  # noqa: E402
from normint import continuity as ncont  # noqa: E402
from normint import solver as nsolver  # noqa: E402
from normint.geometry import CameraIntrinsics, NormalMap  # noqa: E402

OUT = os.path.join(HERE, "full")
STRIDE = 64

CASES = {
    "C1": (lambda: scenes.config1(), None),
    "C2": (lambda: scenes.config2(), None),
    "C3": (lambda: scenes.config3(), None),
    "C4": (lambda: scenes.config4(), 5),
    "C5_00": (lambda: scenes.config5_map(0), None),
    "C5_21": (lambda: scenes.config5_map(21), None),
    "C5_42": (lambda: scenes.config5_map(42), None),
    "C5_63": (lambda: scenes.config5_map(63), None),
}


def normals_digest(n32: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(n32, np.float32).tobytes()).hexdigest()[:16]


def run(name):
    factory, merge = CASES[name]
    sc = factory()
    n32, mask = sc.normals, sc.mask
    settings = nsolver.SolveSettings(freq_merging=merge, worker_count=1)
    weights = ncont.WeightParams()
    nm = NormalMap.create(n32.astype(np.float64), mask)
    cam = CameraIntrinsics(*sc.intrinsics())
    t0 = time.perf_counter()
    res = normint.run_pipeline(nm, cam, float(np.deg2rad(3.5)), settings, weights, 8, "milano")
    secs = time.perf_counter() - t0
    lab0 = res.partition0.labels
    valid = lab0 >= 0
    z = res.log_depth.values.ravel()
    f = res.filled.values.ravel()
    diff = (z - f)[valid]
    cnt = np.bincount(lab0[valid], minlength=res.partition0.component_count)
    scales = np.bincount(lab0[valid], weights=diff, minlength=res.partition0.component_count)
    scales = scales / np.maximum(cnt, 1)
    vidx = np.flatnonzero(mask.ravel())
    sample = vidx[::STRIDE].astype(np.int32)
    rec = [{k: v for k, v in r.items() if k != "wall_ms"} for r in res.records]
    capped = any(w.startswith("iteration") for w in res.warnings)
    d = dict(
        digest=normals_digest(n32), shape=np.array(mask.shape, np.int32),
        labels0=lab0.astype(np.int32).reshape(mask.shape),
        count0=res.partition0.component_count,
        labels=res.partition.labels.astype(np.int32).reshape(mask.shape),
        count=res.partition.component_count,
        iterations=res.iterations, energies=np.array(res.energies),
        records=json.dumps(rec), warnings=json.dumps(res.warnings),
        scales=scales, sample_idx=sample, log_depth_s=z[sample], filled_s=f[sample],
        mean_depth=float(np.mean(np.exp(z[valid]))), scale_cg_capped=capped,
        merge_freq=-1 if merge is None else merge, ref_seconds=secs,
    )
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(f"{name}: {mask.shape} valid={int(mask.sum())} comps={d['count0']}->{d['count']} "
          f"iters={d['iterations']} capped={capped} warnings={len(res.warnings)} {secs:.1f}s",
          flush=True)


def main():
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run(n)


if __name__ == "__main__":
    main()

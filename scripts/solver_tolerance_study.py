"""Would a different (faster-converging) fill solver keep parity?

Runs the CPU oracle twice on the same inputs: with the reference's scipy CG
semantics (rtol 1e-6 from x0 = 0), and with the fill's CG driven to rtol 1e-12
(the limit any tightly converged solver -- multigrid-preconditioned CG, an
on-chip solve -- reaches).  Reports whether labels, outer iterations and
merged partitions agree and the depth error against the north-star bound.

    python scripts/solver_tolerance_study.py [C5|C2|C3s|C4s ...]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import normint_oracle as O  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402
from tests.parity import depth_error  # noqa: E402

CASES = {
    "C5": lambda: scenes.config5_map(0),
    "C2": lambda: scenes.config2(),
    "C3s": lambda: scenes.config3(size=512, cells=32),
    "C4s": lambda: scenes.config4(size=512, cells=128),
}


def run(sc, tight):
    orig = O.conjugate_gradient
    if tight:
        def cg(matvec, b, rtol, maxiter):
            return orig(matvec, b, 1e-12, 20 * maxiter)
        O.conjugate_gradient = cg
    try:
        t = time.perf_counter()
        r = O.run_pipeline(sc.normals.astype(np.float64), sc.mask, sc.intrinsics(),
                           float(np.deg2rad(3.5)),
                           O.Settings(freq_merging=sc.options.get("merge_freq")))
        return r, time.perf_counter() - t
    finally:
        O.conjugate_gradient = orig


for name in sys.argv[1:] or ["C2", "C3s", "C4s", "C5"]:
    sc = CASES[name]()
    a, ta = run(sc, False)
    b, tb = run(sc, True)
    err, bound = depth_error(b.log_depth, a.log_depth, sc.mask, sc.fx)
    ferr, fbound = depth_error(b.filled, a.filled, sc.mask, sc.fx)
    print(f"{name}: valid={int(sc.mask.sum())} comps={a.count0} iters {a.iterations} vs {b.iterations} "
          f"partition_same={np.array_equal(a.labels, b.labels)} "
          f"depth_err={err:.3e} bound={bound:.3e} ratio={err / bound:.3f} "
          f"filled_err={ferr:.3e} ({ta:.1f} s / {tb:.1f} s)", flush=True)

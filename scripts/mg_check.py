"""Multigrid fill vs the oracle's scipy-semantics CG fill on BASELINE-shaped
maps: filled-state error, PCG iterations, level sizes, device time.

    python scripts/mg_check.py [c5] [c3] [c4] [batch N]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import pipeline as P, scenes  # noqa: E402
from oracle import normint_oracle as O  # noqa: E402

THETA = float(np.deg2rad(3.5))


def one(name, sc, oracle=True, merge=None):
    nm = nb.NormalMap.create(sc.normals, sc.mask)
    st = nb.SolveSettings(freq_merging=merge)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), THETA, st)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rep = r.fill_report
    print(f"{name}: step {dt*1e3:.1f} ms fill-loop {rep['cg_ms']:.2f} ms mg {rep.get('mg')} "
          f"iters max {int(r.fill_iterations.max()) if len(r.fill_iterations) else 0} "
          f"outer {r.iterations} warnings {r.warnings[:3]}", flush=True)
    if oracle:
        ref = O.run_pipeline(sc.normals.astype(np.float64), sc.mask, sc.intrinsics(), THETA,
                             O.Settings(freq_merging=merge))
        m = sc.mask
        fe = np.abs(r.filled.values - ref.filled)[m]
        de = np.abs(np.exp(r.log_depth.values[m]) - np.exp(ref.log_depth[m]))
        print(f"   filled max {fe.max():.2e} mean {fe.mean():.2e}; depth mean {de.mean():.2e} "
              f"(bound {1e-4*np.mean(np.exp(ref.log_depth[m])) + 1e-3/sc.fx:.2e}); "
              f"outer {r.iterations} vs {ref.iterations}; labels "
              f"{np.array_equal(r.partition0.labels, ref.labels0)}", flush=True)


def main():
    args = sys.argv[1:] or ["small", "c5"]
    if "small" in args:
        one("c4_96", scenes.config4(3, size=96, cells=14), merge=5)
        one("c5_48", scenes.config5_map(0, size=48, cells=5))
        one("c2_96x80", scenes.config2(1, h=80, w=96, f=580.0, frac=0.4))
        one("C1", scenes.config1())
        one("C2", scenes.config2())
    if "c5" in args:
        one("c5_map0", scenes.config5_map(0))
    if "c3" in args:
        one("C3", scenes.config3(), oracle=False)
    if "c4" in args:
        one("C4", scenes.config4(), oracle=False, merge=5)
    if "batch" in args:
        n = int(args[args.index("batch") + 1])
        scs = [scenes.config5_map(i) for i in range(n)]
        nm = nb.NormalMap.create(np.stack([s.normals for s in scs]), np.stack([s.mask for s in scs]))
        intr = [nb.CameraIntrinsics(*s.intrinsics()) for s in scs]
        prev = None
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rs = nb.run_pipeline_batch(nm, intr, THETA)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            its = [int(r.fill_iterations.max()) for r in rs]
            filled = torch.cat([r.filled.values_t for r in rs])
            same = None if prev is None else bool(torch.equal(prev, filled))
            prev = filled
            print(f"batch {n}: step {dt*1e3:.1f} ms fill-loop {rs[0].fill_report['cg_ms']:.2f} ms "
                  f"mg {rs[0].fill_report.get('mg')} -> {n * 1048576 / dt / 1e6:.1f} M px/s "
                  f"fill iters max {max(its)} mean {np.mean(its):.1f} rerun-identical {same}",
                  flush=True)


if __name__ == "__main__":
    main()

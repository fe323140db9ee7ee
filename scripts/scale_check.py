"""Large / unusual configurations through run_pipeline: C3 and C4 at full size
and a theta_c = None map (one component per pixel), with wall times."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402


def run(name, sc, theta, merge=None):
    nm = nb.NormalMap.create(sc.normals, sc.mask)
    st = nb.SolveSettings(freq_merging=merge)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), theta, st)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
    rec = {x["stage"]: x["wall_ms"] for x in r.records if "stage" in x}
    print(f"{name}: {ms:.1f} ms valid={int(sc.mask.sum())} comps {r.partition0.component_count}->"
          f"{r.partition.component_count} iters={r.iterations} fill={rec['fill']:.1f} ms "
          f"max_cg={int(r.fill_iterations.max()) if len(r.fill_iterations) else 0} "
          f"warnings={len(r.warnings)}", flush=True)


def records_c4():
    sc = scenes.CONFIGS["C4"]()
    nm = nb.NormalMap.create(sc.normals, sc.mask)
    st = nb.SolveSettings(freq_merging=5)
    for rep in range(2):
        r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), float(np.deg2rad(3.5)), st)
    for x in r.records:
        print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in x.items()
               if k not in ("z_digest_before", "z_digest_after")})


if __name__ == "__main__" and sys.argv[1:2] == ["records"]:
    records_c4()
elif __name__ == "__main__":
    which = sys.argv[1:] or ["none256", "C3", "C4"]
    if "none256" in which:
        run("C1 theta=None", scenes.CONFIGS["C1"](), None)
    if "C3" in which:
        run("C3", scenes.CONFIGS["C3"](), float(np.deg2rad(3.5)))
    if "C4" in which:
        run("C4 merge5", scenes.CONFIGS["C4"](), float(np.deg2rad(3.5)), 5)

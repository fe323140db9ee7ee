"""Host-side stage times of run_pipeline from its diagnostics records (the
`wall_ms` of each stage / iteration record), for one config:

    python scripts/stage_times.py C1 [reps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sc = scenes.CONFIGS[name]()
nm_args = (sc.normals, sc.mask)
intr = nb.CameraIntrinsics(*sc.intrinsics())
st = nb.SolveSettings(freq_merging=sc.options.get("merge_freq"))
theta = float(np.deg2rad(3.5))
for rep in range(reps):
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    t0 = time.perf_counter()
    nm = nb.NormalMap.create(*nm_args)
    t1 = time.perf_counter()
    r = nb.run_pipeline(nm, intr, theta, st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    stages = {x["stage"]: x["wall_ms"] for x in r.records if "stage" in x}
    loop = sum(x["wall_ms"] for x in r.records if "t" in x)
    print(f"rep {rep}: create {1e3 * (t1 - t0):.2f} ms, run {1e3 * (t2 - t1):.2f} ms, "
          f"launches {_lib.launch_count() - l0}, iterations {r.iterations}; stages "
          + ", ".join(f"{k} {v:.2f}" for k, v in stages.items()) + f", loop {loop:.2f}",
          flush=True)

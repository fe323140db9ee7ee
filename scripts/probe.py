"""Quick GPU probe: run configs through run_pipeline, print timings/stats."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

cfgs = sys.argv[1:] or ["C1", "C2"]
for cfg in cfgs:
    t = time.time()
    if cfg.startswith("C3s"):
        sc = scenes.config3(size=int(cfg[3:]))
    else:
        sc = scenes.CONFIGS[cfg]()
    gen = time.time() - t
    theta = float(np.deg2rad(3.5))
    st = nb.SolveSettings(freq_merging=sc.options.get("merge_freq"))
    prev = None
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.time()
        nm = nb.NormalMap.create(sc.normals, sc.mask)
        r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), theta, st)
        torch.cuda.synchronize()
        el = time.time() - t
        stages = {x.get("stage", "it"): round(x["wall_ms"], 1) for x in r.records if "stage" in x}
        it_ms = sum(x["wall_ms"] for x in r.records if "t" in x)
        fi = r.fill_iterations
        print(f"{cfg} rep{rep}: gen {gen:.1f}s total {el*1e3:.1f} ms valid {sc.valid_count} "
              f"comps {r.partition0.component_count}->{r.partition.component_count} outer {r.iterations} "
              f"stages {stages} outer_ms {it_ms:.1f} fill_iters max {fi.max() if len(fi) else 0} "
              f"warnings {len(r.warnings)}", flush=True)
        cur = r.log_depth.values.copy()
        if prev is not None:
            print(f"{cfg}: bit-identical rerun: {np.array_equal(prev, cur)}", flush=True)
        prev = cur

"""Warm-up + one profiled run_pipeline of a single-map config, for ncu captures:

    ncu ... -k regex:scale_fused -s 3 -c 1 python scripts/profile_cfg.py C1
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
sc = scenes.CONFIGS[name]()
intr = nb.CameraIntrinsics(*sc.intrinsics())
st = nb.SolveSettings(freq_merging=sc.options.get("merge_freq"))
for _ in range(2):
    r = nb.run_pipeline(nb.NormalMap.create(sc.normals, sc.mask), intr, float(np.deg2rad(3.5)), st)
    torch.cuda.synchronize()
print(r.iterations, r.partition0.component_count, r.records[-1])

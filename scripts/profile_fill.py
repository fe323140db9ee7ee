"""Run the batched pipeline on a small C5-like batch twice (the second run is
the one to capture under ncu: -k regex:fill_cg -s 1 -c 1)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402

nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
maps = [scenes.config5_map(i) for i in range(nmaps)]
n = torch.from_numpy(np.stack([m.normals for m in maps])).cuda()
mk = torch.from_numpy(np.stack([m.mask for m in maps])).cuda()
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
for rep in range(2):
    nm = nb.NormalMap.create(n, mk)
    res = nb.run_pipeline_batch(nm, intr, float(np.deg2rad(3.5)))
    torch.cuda.synchronize()
    rep_ = _lib.fill_report()
    print(rep, rep_, "GB/s", 45 * rep_["px_iters"] / (rep_["cg_ms"] * 1e-3) / 1e9, flush=True)

"""One warm-up + one profiled batched run of N C5 maps (for ncu launch lists /
--set full captures of the multigrid fill kernels)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
maps = [scenes.config5_map(i) for i in range(nmaps)]
n = torch.from_numpy(np.stack([m.normals for m in maps])).cuda()
mk = torch.from_numpy(np.stack([m.mask for m in maps])).cuda()
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
for rep in range(2):
    nm = nb.NormalMap.create(n, mk)
    res = nb.run_pipeline_batch(nm, intr, float(np.deg2rad(3.5)))
    torch.cuda.synchronize()
    print(rep, res[0].fill_report, flush=True)

"""Trace one unit's PCG scalars on C5 map 0 (NI_MG_TRACE=<unit>)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

sc = scenes.config5_map(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
nm = nb.NormalMap.create(sc.normals, sc.mask)
r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), float(np.deg2rad(3.5)))
torch.cuda.synchronize()
print("fill iters", r.fill_iterations.tolist(), "sizes", r.partition0.sizes.tolist())
print("warnings", r.warnings)

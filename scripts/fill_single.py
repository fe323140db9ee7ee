"""Fill report for a single large map (C3 or C4) through run_pipeline."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
sc = scenes.CONFIGS[cfg]()
nm = nb.NormalMap.create(sc.normals, sc.mask)
for rep in range(2):
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), float(np.deg2rad(3.5)))
    torch.cuda.synchronize()
    f = _lib.fill_report()
    print(f"{cfg} rep{rep} cg_ms={f['cg_ms']:.1f} px_iters={f['px_iters']:.3e} max_iters={f['max_iters']} "
          f"items={f['ntiles']} GB/s={37 * f['px_iters'] / (f['cg_ms'] * 1e-3) / 1e9:.1f}", flush=True)

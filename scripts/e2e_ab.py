"""e2e stream A/B: ms per step of run_pipeline_stream over the 64-map C5 batch
for several read-back CTA counts (0 = copy-engine read-back) and stream
priorities, interleaved.

    python scripts/e2e_ab.py [ctas[:priority[:upload_ctas]] ...]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import pipeline, scenes  # noqa: E402

variants = [tuple(int(y) for y in (x.split(":") + ["-1", "0"])[:3]) for x in sys.argv[1:]] or [(2, -1, 0)]
maps = [scenes.config5_map(i) for i in range(64)]
n = torch.from_numpy(np.stack([m.normals for m in maps]).astype(np.float32)).pin_memory()
k = torch.from_numpy(np.stack([m.mask for m in maps])).pin_memory()
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
st = nb.SolveSettings()
theta = float(np.deg2rad(3.5))


def run(steps):
    for _ in nb.run_pipeline_stream(((n, k) for _ in range(steps)), intr, theta, st):
        pass


run(3)
for rep in range(3):
    for v, prio, up in variants:
        pipeline._D2H_CTAS = v
        pipeline._D2H_PRIORITY = prio
        pipeline._H2D_CTAS = up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run(10)
        torch.cuda.synchronize()
        print(f"rep {rep} read-back ctas {v} priority {prio} upload ctas {up}: {1e3 * (time.perf_counter() - t0) / 10:.2f} ms/step", flush=True)

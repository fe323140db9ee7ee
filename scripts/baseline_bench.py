"""Pixel-level baseline vs the component pipeline on C5 maps (first N):
wall time of run_pixel_baseline_batch and run_pipeline_batch on the same
batch (second run of each; the first warms up)."""
import concurrent.futures as cf
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402


def gen(i):
    m = scenes.config5_map(i)
    return m.normals, m.mask, m.intrinsics()


if __name__ == "__main__":
    nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    with cf.ProcessPoolExecutor(max_workers=min(nmaps, os.cpu_count() or 1)) as ex:
        maps = list(ex.map(gen, range(nmaps)))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda()
    mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    for name, fn in (("pipeline", lambda nm: nb.run_pipeline_batch(nm, intr, float(np.deg2rad(3.5)))),
                     ("pixel_baseline", lambda nm: nb.run_pixel_baseline_batch(nm, intr))):
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fn(nb.NormalMap.create(n, mk))
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
        its = [r.iterations for r in res]
        print(f"{name}: maps={nmaps} {ms:.1f} ms  outer iterations max {max(its)} mean {np.mean(its):.1f}",
              flush=True)

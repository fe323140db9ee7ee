"""Robustness / throughput of run_pipeline_batch on other batch shapes:
    python scripts/scale_shapes.py  ->  one line per shape (maps x size, ms, valid px/s, fill GB/s)"""
import concurrent.futures as cf
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402


def gen(args):
    i, size, cells = args
    s = scenes.voronoi_ortho(f"m{i}", size, size, cells, 500 + i, 0.2)
    return s.normals, s.mask, s.intrinsics()


for nmaps, size, cells in [(16, 2048, 64), (4, 4096, 128), (256, 256, 4), (1024, 128, 3)]:
    with cf.ProcessPoolExecutor(16) as ex:
        maps = list(ex.map(gen, [(i, size, cells) for i in range(nmaps)]))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda()
    mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, float(np.deg2rad(3.5)))
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
    f = _lib.fill_report()
    px = int(mk.sum())
    print(f"{nmaps} x {size}^2: {ms:.1f} ms, {px / ms / 1e3:.1f} M px/s, fill {f['cg_ms']:.1f} ms "
          f"= {37 * f['px_iters'] / (f['cg_ms'] * 1e-3) / 1e9:.0f} GB/s, outer iters max "
          f"{max(r.iterations for r in res)}", flush=True)
    del n, mk, res
    torch.cuda.empty_cache()

"""cProfile of run_pipeline_batch on the C5 batch (second run): where the host
time of the outer loop goes (ctypes calls, read-back waits, bookkeeping)."""
import concurrent.futures as cf
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402


def gen(i):
    m = scenes.config5_map(i)
    return m.normals, m.mask, m.intrinsics()


if __name__ == "__main__":
    nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    with cf.ProcessPoolExecutor(max_workers=min(nmaps, os.cpu_count() or 1)) as ex:
        maps = list(ex.map(gen, range(nmaps)))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda()
    mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, float(np.deg2rad(3.5)))
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, float(np.deg2rad(3.5)))
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)

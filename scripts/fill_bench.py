"""Fill-kernel throughput on a C5-like batch (first N maps), DRAM-resident."""
import concurrent.futures as cf
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402


def gen(i):
    m = scenes.config5_map(i)
    return m.normals, m.mask, m.intrinsics()


if __name__ == "__main__":
    nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    with cf.ProcessPoolExecutor(max_workers=min(nmaps, os.cpu_count() or 1)) as ex:
        maps = list(ex.map(gen, range(nmaps)))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda()
    mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    for rep in range(2):
        nm = nb.NormalMap.create(n, mk)
        res = nb.run_pipeline_batch(nm, intr, float(np.deg2rad(3.5)))
        torch.cuda.synchronize()
        r = _lib.fill_report()
        print(f"minb={os.environ.get('NI_FILL_MINB', '4')} rep{rep} maps={nmaps} cg_ms={r['cg_ms']:.1f} "
              f"px_iters={r['px_iters']:.3e} max_iters={r['max_iters']} grid={r['grid']} items={r['ntiles']} "
              f"GB/s={37 * r['px_iters'] / (r['cg_ms'] * 1e-3) / 1e9:.1f}", flush=True)

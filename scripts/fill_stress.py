"""Scheduler stress: the batched fill under every mailbox depth / pairing mode,
repeated, on a C5-like batch; each run must finish (per-run timeout by the
caller) and reproduce the first run's fill bit for bit.

    timeout 900 python scripts/fill_stress.py [nmaps] [reps]
"""
import concurrent.futures as cf
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402
from paper_2510_11508_b200.pipeline import _coefficients, _components, _fill, _Grid  # noqa: E402,F401


def gen(i):
    m = scenes.config5_map(i)
    return m.normals, m.mask, m.intrinsics()


if __name__ == "__main__":
    nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    with cf.ProcessPoolExecutor(max_workers=min(nmaps, os.cpu_count() or 1)) as ex:
        maps = list(ex.map(gen, range(nmaps)))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda()
    mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    ref = None
    for mode in [{}, {"NI_FILL_MB": "1"}, {"NI_FILL_MB": "2"}, {"NI_FILL_PAIR": "1"},
                 {"NI_FILL_PAIR": "2", "NI_FILL_MB": "1"}]:
        for k in ("NI_FILL_MB", "NI_FILL_PAIR"):
            os.environ.pop(k, None)
        os.environ.update(mode)
        for r in range(reps):
            t = time.perf_counter()
            res = nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, float(np.deg2rad(3.5)))
            torch.cuda.synchronize()
            f = _lib.fill_report()
            z = torch.cat([x.filled.values_t for x in res])
            if ref is None:
                ref = z.clone()
            same = bool(torch.equal(ref, z)) if "NI_FILL_PAIR" not in mode else None
            print(f"{mode or 'default'} rep {r}: fill {f['cg_ms']:.1f} ms, step "
                  f"{(time.perf_counter() - t) * 1e3:.0f} ms, filled identical to first run: {same}",
                  flush=True)

"""Per-stage wall times of run_pipeline_batch on the C5 batch (first N maps),
from the records the pipeline writes (second run; the first warms up)."""
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
    nmaps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    with cf.ProcessPoolExecutor(max_workers=min(nmaps, os.cpu_count() or 1)) as ex:
        maps = list(ex.map(gen, range(nmaps)))
    n = torch.from_numpy(np.stack([m[0] for m in maps])).cuda()
    mk = torch.from_numpy(np.stack([m[1] for m in maps])).cuda()
    intr = [nb.CameraIntrinsics(*m[2]) for m in maps]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nm = nb.NormalMap.create(n, mk)
        res = nb.run_pipeline_batch(nm, intr, float(np.deg2rad(3.5)))
        torch.cuda.synchronize()
        total = (time.perf_counter() - t0) * 1e3
    r0 = res[0].records
    st = {r["stage"]: r["wall_ms"] for r in r0 if "stage" in r}
    outer = sum(r["wall_ms"] for res_m in res for r in res_m.records if "t" in r)
    iters = [res_m.iterations for res_m in res]
    print(f"maps={nmaps} total={total:.1f} ms components={st['form_components']:.1f} "
          f"coefficients={st['edge_coefficients']:.1f} fill={st['fill']:.1f} "
          f"(cg {res[0].fill_report['cg_ms']:.1f}) outer_loops={outer:.1f} "
          f"(outer iterations {sum(iters)}, mean {np.mean(iters):.1f}) done_at={st['done']:.1f}")

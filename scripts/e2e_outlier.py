"""Why some e2e stream runs are 10-16 ms per step slower than the others: per run
of 10 steps, ms per step, the largest pinned read-back allocation and the GC
activity.

    python scripts/e2e_outlier.py [runs] [nogc|freeze]
"""
import gc
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import pipeline, scenes  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 12
maps = [scenes.config5_map(i) for i in range(64)]
n = torch.from_numpy(np.stack([m.normals for m in maps]).astype(np.float32)).pin_memory()
k = torch.from_numpy(np.stack([m.mask for m in maps])).pin_memory()
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
st = nb.SolveSettings()
theta = float(np.deg2rad(3.5))


gc_log = []
_t = {}


def _gc_cb(phase, info):
    if phase == "start":
        _t["t"] = time.perf_counter()
    else:
        gc_log.append((info["generation"], 1e3 * (time.perf_counter() - _t["t"])))


gc.callbacks.append(_gc_cb)
NOGC = len(sys.argv) > 2 and sys.argv[2] == "nogc"
FREEZE = len(sys.argv) > 2 and sys.argv[2] == "freeze"


def run(steps):
    per = []
    t = time.perf_counter()
    for _ in nb.run_pipeline_stream(((n, k) for _ in range(steps)), intr, theta, st):
        t2 = time.perf_counter()
        per.append(1e3 * (t2 - t))
        t = t2
    return per


run(3)
if FREEZE:
    gc.collect()
    gc.freeze()
for r in range(runs):
    torch.cuda.synchronize()
    g0 = sum(s["collections"] for s in gc.get_stats())
    pipeline._PIN_ALLOC_MS.clear()
    gc_log.clear()
    if NOGC:
        gc.collect()
        gc.disable()
    t0 = time.perf_counter()
    per = run(10)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0) / 10
    if NOGC:
        gc.enable()
    print(f"run {r}: {ms:6.2f} ms/step, max pinned alloc {max(pipeline._PIN_ALLOC_MS):7.2f} ms, "
          f"gc collections {sum(s['collections'] for s in gc.get_stats()) - g0}, "
          f"longest gc pauses (gen, ms) {sorted(gc_log, key=lambda g: -g[1])[:3]}, "
          f"yield gaps {' '.join(f'{x:.0f}' for x in per)}", flush=True)

"""Where the e2e stream's extra time goes: ms per step of run_pipeline_stream
over the 64-map C5 batch with the upload and / or the read-back switched off,
against the device-resident step, interleaved.

    python scripts/e2e_split.py [steps]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import _lib, scenes  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
maps = [scenes.config5_map(i) for i in range(64)]
n = torch.from_numpy(np.stack([m.normals for m in maps]).astype(np.float32)).pin_memory()
k = torch.from_numpy(np.stack([m.mask for m in maps])).pin_memory()
n_dev, k_dev = n.cuda(), k.cuda()
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
st = nb.SolveSettings()
theta = float(np.deg2rad(3.5))
lib = _lib.load()
real_copy = lib.ni_copy_to_host


def run(upload, readback):
    lib.ni_copy_to_host = real_copy if readback else (lambda *a: 0)
    src = (n, k) if upload else (n_dev, k_dev)
    for _ in nb.run_pipeline_stream((src for _ in range(steps)), intr, theta, st):
        pass
    lib.ni_copy_to_host = real_copy


def device_steps():
    for _ in range(steps):
        nb.run_pipeline_batch(nb.NormalMap.create(n_dev, k_dev), intr, theta, st)


run(True, True)
device_steps()
for rep in range(2):
    for name, fn in (("device-resident", device_steps),
                     ("stream, no copies", lambda: run(False, False)),
                     ("stream, upload only", lambda: run(True, False)),
                     ("stream, read-back only", lambda: run(False, True)),
                     ("stream, both", lambda: run(True, True))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        print(f"rep {rep} {name}: {1e3 * (time.perf_counter() - t0) / steps:.2f} ms/step",
              flush=True)

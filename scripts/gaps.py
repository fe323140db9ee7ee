"""GPU idle time inside one device-resident C5 step (torch.profiler / CUPTI):
the union of kernel + memcpy intervals against the step's span, and the
largest gaps with the kernels on either side.

    python scripts/gaps.py [maps]
"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
STREAM = len(sys.argv) > 2 and sys.argv[2] == "stream"  # profile 4 steps of run_pipeline_stream
maps = [scenes.config5_map(i) for i in range(B)]
n = torch.from_numpy(np.stack([m.normals for m in maps]).astype(np.float32)).cuda()
k = torch.from_numpy(np.stack([m.mask for m in maps])).cuda()
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
st = nb.SolveSettings()
theta = float(np.deg2rad(3.5))


n_pin, k_pin = n.cpu().pin_memory(), k.cpu().pin_memory()


def step():
    if STREAM:
        for _ in nb.run_pipeline_stream(((n_pin, k_pin) for _ in range(4)), intr, theta, st):
            pass
        return None
    return nb.run_pipeline_batch(nb.NormalMap.create(n, k), intr, theta, st)


for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
      and not e.name.startswith("void ni::d2h_mapped") and "HtoD (Pinned" not in e.name]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
span = iv[-1][1] - iv[0][0]
busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
gaps = []
last = iv[0][2]
for s, e, name in iv[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, last[:50], name[:50]))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    if e >= cur_e:
        last = name
busy += cur_e - cur_s
print(f"span {span / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, idle {(span - busy) / 1e3:.2f} ms, "
      f"{len(iv)} device events, {len(gaps)} gaps")
# copies: how many, and how long they take (control reads / uploads queue behind
# bulk transfers on the same link direction)
import collections  # noqa: E402
cp = collections.defaultdict(lambda: [0, 0.0])
for s_, e_, name in iv:
    if name.startswith("Mem"):
        cp[name][0] += 1
        cp[name][1] += e_ - s_
for name, (cnt, tot_us) in sorted(cp.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:45s} {cnt:5d} x {tot_us / max(cnt, 1):8.1f} us = {tot_us / 1e3:7.2f} ms")
gaps.sort(reverse=True)
tot = sum(g[0] for g in gaps)
print(f"gaps > 50 us: {sum(g[0] for g in gaps if g[0] > 50) / 1e3:.2f} ms; "
      f"gaps 10-50 us: {sum(g[0] for g in gaps if 10 < g[0] <= 50) / 1e3:.2f} ms; "
      f"< 10 us: {sum(g[0] for g in gaps if g[0] <= 10) / 1e3:.2f} ms (total {tot / 1e3:.2f})")
for g in gaps[:40]:
    print(f"{g[0]:8.1f} us  after {g[1]:50s} before {g[2]}")

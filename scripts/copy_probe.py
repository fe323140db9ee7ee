"""Does a large pinned host<->device transfer on a side stream delay the small
control copies (.cpu() / .to(dev)) of the compute stream?  Prints the latency
of small D2H / H2D copies alone, under a big H2D, under a big D2H, and under
the same big transfers done by an SM copy kernel over mapped host memory.

    python scripts/copy_probe.py
"""
import time

import torch

dev = torch.device("cuda:0")
N = 872 * 2**20
host_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
host_out = torch.empty(537 * 2**20, dtype=torch.uint8, pin_memory=True)
dev_in = torch.empty(N, dtype=torch.uint8, device=dev)
dev_out = torch.empty(host_out.numel(), dtype=torch.uint8, device=dev)
small_d = torch.zeros(64, dtype=torch.float64, device=dev)
side = torch.cuda.Stream(dev)


def small_lat(reps=20):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        small_d.cpu()
        t1 = time.perf_counter()
        torch.ones(16, dtype=torch.int32).to(dev)
        torch.cuda.current_stream().synchronize()
        t2 = time.perf_counter()
        t.append((1e3 * (t1 - t0), 1e3 * (t2 - t1)))
    d2h = sorted(x[0] for x in t)[reps // 2]
    h2d = sorted(x[1] for x in t)[reps // 2]
    return f"small d2h {d2h:.3f} ms, small h2d {h2d:.3f} ms"


def big_h2d():
    with torch.cuda.stream(side):
        dev_in.copy_(host_in, non_blocking=True)


def big_d2h():
    with torch.cuda.stream(side):
        host_out.copy_(dev_out, non_blocking=True)


torch.cuda.synchronize()
print("alone:", small_lat(), flush=True)
for name, fn in (("big h2d", big_h2d), ("big d2h", big_d2h)):
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        first = small_lat(1)
        side.synchronize()
        t1 = time.perf_counter()
        print(f"under {name}: first {first}; big transfer {1e3 * (t1 - t0):.1f} ms", flush=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
big_h2d()
side.synchronize()
print(f"h2d alone {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
t0 = time.perf_counter()
big_d2h()
side.synchronize()
print(f"d2h alone {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)

# the same read-back by the SM kernel over mapped pinned memory (ni_copy_to_host)
import ctypes as C  # noqa: E402
import sys  # noqa: E402

sys.path.insert(0, ".")
from paper_2510_11508_b200 import _lib  # noqa: E402

lib = _lib.load()
hi = torch.cuda.Stream(dev, priority=-1)
for ctas in (16, 32, 64, 148):
    def kern_d2h():
        _lib.check(lib.ni_copy_to_host(C.c_void_p(dev_out.data_ptr()),
                                       C.c_void_p(host_out.data_ptr()), dev_out.numel(), ctas,
                                       C.c_void_p(hi.cuda_stream)), "copy")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kern_d2h()
        first = small_lat(1)
        hi.synchronize()
        t1 = time.perf_counter()
        print(f"under kernel d2h ({ctas} CTAs): first {first}; big transfer "
              f"{1e3 * (t1 - t0):.1f} ms", flush=True)

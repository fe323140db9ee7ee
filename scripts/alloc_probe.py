"""Host cost of the fill's workspace allocation path (why ~0.35 ms pass between the last
torch kernel and ni_fill_mg's first memset on the C5 batch)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_11508_b200 import _lib  # noqa: E402

lib = _lib.load()
B, H, W = 64, 1024, 1024
t = time.perf_counter()
n = _lib.size_query(lib.ni_fill_mg_workspace_size, B, H, W, 8, 1100)
print(f"size query: {1e6 * (time.perf_counter() - t):.0f} us, {n / 1e9:.2f} GB")
for rep in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ws = torch.empty(n, dtype=torch.uint8, device="cuda")
    t1 = time.perf_counter()
    z = torch.empty(B * H * W, dtype=torch.float64, device="cuda")
    t2 = time.perf_counter()
    it = torch.zeros(1100, dtype=torch.int32, device="cuda")
    t3 = time.perf_counter()
    del ws, z, it
    t4 = time.perf_counter()
    print(f"rep {rep}: empty(ws) {1e6 * (t1 - t):.0f} us, empty(z) {1e6 * (t2 - t1):.0f} us, "
          f"zeros {1e6 * (t3 - t2):.0f} us, del {1e6 * (t4 - t3):.0f} us")

"""Map-level data parallelism for batched runs (BASELINE.json config 5).

Independent normal maps are split across ranks in contiguous blocks; there is
no data-path collective.  The only collectives are the result aggregation of
bench.py: a sum of valid pixels and a max of the per-rank device step time
(the whole job takes as long as its slowest rank).  Works with any
torch.distributed backend (NCCL on the GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def map_range(rank: int, world: int, nmaps: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of maps owned by `rank`."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * nmaps // world, (rank + 1) * nmaps // world


def aggregate(valid_local: int, ms_local: float, device=None) -> tuple[int, float]:
    """(sum of valid pixels, max of step milliseconds) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return int(valid_local), float(ms_local)
    dev = device if device is not None else torch.device("cpu")
    v = torch.tensor([float(valid_local)], dtype=torch.float64, device=dev)
    t = torch.tensor([float(ms_local)], dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return int(v.item()), float(t.item())

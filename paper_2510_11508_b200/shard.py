"""Map-level data parallelism for batched runs (BASELINE.json config 5).

Independent normal maps are split across ranks in contiguous blocks; there is
no data-path collective.  The only collective is the result gather of
bench.py: one all_gather of every rank's (valid pixels, device step ms, outer
iterations, maps) row, from which rank 0 forms the whole-job numbers (valid
pixels summed, the step taking as long as its slowest rank).  Works with any
torch.distributed backend (NCCL over NVLink on the GPUs, gloo in the CPU
tests).
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


STAT_FIELDS = ("valid_px", "ms", "outer_iters", "maps")


def gather_stats(valid_px: int, ms: float, outer_iters: int, maps: int, device=None) -> list[dict]:
    """all_gather of each rank's step statistics; returns one dict per rank
    (rank order).  A single process returns its own row."""
    row = [float(valid_px), float(ms), float(outer_iters), float(maps)]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        rows = [row]
    else:
        dev = device if device is not None else torch.device("cpu")
        mine = torch.tensor(row, dtype=torch.float64, device=dev)
        out = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
        dist.all_gather(out, mine)
        rows = [o.cpu().tolist() for o in out]
    return [dict(zip(STAT_FIELDS, r)) for r in rows]


def whole_job(stats: list[dict]) -> tuple[int, float]:
    """(valid pixels over all ranks, the slowest rank's step ms)."""
    return int(sum(s["valid_px"] for s in stats)), float(max(s["ms"] for s in stats))

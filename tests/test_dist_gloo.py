"""World-size-2 test of the map sharding and result aggregation used by
bench.py, on the CPU with the gloo backend (NCCL stands in on the GPUs)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2510_11508_b200.shard import map_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nmaps, q):
    import torch.distributed as dist

    from paper_2510_11508_b200.shard import aggregate, map_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = map_range(rank, world, nmaps)
    valid_local = sum(1000 + i for i in range(lo, hi))
    ms_local = 10.0 * (rank + 1)
    total, ms = aggregate(valid_local, ms_local)
    q.put((rank, lo, hi, total, ms))
    dist.destroy_process_group()


def test_map_range_partitions():
    for world in (1, 2, 4, 8):
        got = [map_range(r, world, 64) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == 64
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        assert all(hi - lo == 64 // world for lo, hi in got)
    with pytest.raises(ValueError):
        map_range(2, 2, 8)


def test_two_rank_gloo_aggregation():
    world, nmaps = 2, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nmaps, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect_total = sum(1000 + i for i in range(nmaps))
    assert [o[1:3] for o in out] == [(0, 5), (5, 10)]
    for _, _, _, total, ms in out:
        assert total == expect_total
        assert ms == 20.0  # the slowest rank


def test_gather_stats_single_process():
    from paper_2510_11508_b200.shard import gather_stats, whole_job

    st = gather_stats(123, 4.5, 7, 2)
    assert st == [{"valid_px": 123.0, "ms": 4.5, "outer_iters": 7.0, "maps": 2.0}]
    assert whole_job(st) == (123, 4.5)


@pytest.mark.parametrize("scaling,maps,per_rank", [("weak", 2, [2, 2]), ("strong", 4, [2, 2])])
def test_bench_launcher_two_ranks_gloo(scaling, maps, per_rank):
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself under
    torch.distributed.run; the ranks take their maps (weak: each its own
    batch; strong: halves of one batch), all_gather their stats and rank 0
    alone prints the whole-job line (gloo, no GPU work)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--maps", str(maps), "--scaling", scaling, "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    ranks = line["config"]["per_rank"]
    assert [r["maps"] for r in ranks] == per_rank
    assert line["config"]["maps_total"] == sum(per_rank)
    assert line["config"]["valid_px_total"] == sum(r["valid_px"] for r in ranks)

"""Benchmark: valid pixels/s of the component normal-integration hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step is one pass of the hot path (``run_pipeline`` semantics: normalise ->
components -> coefficients -> batched fill -> relative-scale loop with
merges -> gauge) over one batch of synthetic normal maps.  The default
workload is BASELINE.json config 5: 64 independent 1024x1024 orthographic
maps (seeds 100..163, 16 Voronoi cells), split across ranks by map (strong
scaling: the 64 maps are fixed, each rank takes a contiguous block).

* ``value``: valid px/s with the normals already resident in HBM; whole-job
  = all ranks' valid pixels / max-over-ranks device time of a step.
* ``e2e``: the same through the public API from pinned HOST normals, with
  the host->device copy of the normals+mask and the device->host copy of the
  log-depth inside the timed region.
* ``roofline``: the dominant kernel (the persistent batched CG,
  ``fill_cg_kernel``), algorithmic bytes per launch = 37 B x (component
  size x CG iterations, summed) / its CUDA-event duration.
* ``cpu_baseline``: the CPU oracle port (oracle/normint_oracle.py, a numpy
  restatement of the reference) on one map of the same batch, rank 0, N=1.

``--impl reference`` times that oracle port alone on the host cores (one
process per core, one map per process per step) and prints the same line
with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_PX_ITER = 37  # paper_2510_11508_b200/csrc/ni_fill.cu header (single-sweep CG)
# canonical bytes per px-iteration of a two-sweep PCG at 8-conn
# (56 + 4 K_f); the single-sweep kernel needs only BYTES_PER_PX_ITER of them.
SURVEY_BYTES_PER_PX_ITER = 72
SURVEY_PEAK_GBS = 8000.0  # SURVEY.md 8(d) north-star denominator
THETA_DEG = 3.5


# --------------------------------------------------------------- workloads


def _gen_c5(i):
    from paper_2510_11508_b200 import scenes
    s = scenes.config5_map(i)
    return s.normals, s.mask, s.intrinsics()


def _gen_cfg(name):
    from paper_2510_11508_b200 import scenes
    s = scenes.CONFIGS[name]()
    return s.normals, s.mask, s.intrinsics(), s.options.get("merge_freq")


def make_workload(config, rank, world, nmaps):
    """Return (normals (B,H,W,3) f32, masks (B,H,W) bool, intrinsics list,
    merge_freq, description, total maps)."""
    if config == "C5":
        from paper_2510_11508_b200.shard import map_range
        lo, hi = map_range(rank, world, nmaps)
        idx = list(range(lo, hi))
        import concurrent.futures as cf
        workers = max(1, min(len(idx), (os.cpu_count() or 2) // max(1, world)))
        if workers > 1:
            with cf.ProcessPoolExecutor(max_workers=workers) as ex:
                maps = list(ex.map(_gen_c5, idx))
        else:
            maps = [_gen_c5(i) for i in idx]
        normals = np.stack([m[0] for m in maps])
        masks = np.stack([m[1] for m in maps])
        intr = [m[2] for m in maps]
        desc = f"C5: {nmaps} x 1024x1024 orthographic maps (seeds 100..{99 + nmaps}), 16 Voronoi cells"
        return normals, masks, intr, None, desc, nmaps
    n, m, i, mf = _gen_cfg(config)
    return n[None], m[None], [i], mf, f"{config} (paper_2510_11508_b200/scenes.py)", 1


# -------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 4 + k and r[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profile():
    """dram bytes per launch of fill_cg_kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "fill_cg_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------------ our arm


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2510_11508_b200 as nb
    from paper_2510_11508_b200 import _lib

    normals_h, masks_h, intr_t, merge_freq, desc, total_maps = make_workload(
        args.config, rank, world, args.maps)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _lib.load()
    intr = [nb.CameraIntrinsics(*t) for t in intr_t]
    theta = float(np.deg2rad(THETA_DEG))
    settings = nb.SolveSettings(freq_merging=merge_freq)
    B = normals_h.shape[0]
    valid_local = int(masks_h.sum())

    # device-resident inputs for `value`; pinned host inputs for `e2e`
    n_dev = torch.from_numpy(normals_h).to(dev)
    m_dev = torch.from_numpy(masks_h).to(dev)
    n_pin = torch.from_numpy(normals_h).pin_memory()
    m_pin = torch.from_numpy(masks_h).pin_memory()

    def step_device():
        nm = nb.NormalMap.create(n_dev, m_dev)
        if B == 1:
            return [nb.run_pipeline(nm, intr[0], theta, settings)]
        return nb.run_pipeline_batch(nm, intr, theta, settings)

    def run_e2e(k):
        """k steps through the serving API: every step copies its pinned host
        inputs to the device and reads every map's log-depth back into pinned
        host memory; run_pipeline_stream overlaps the next step's upload and
        the previous step's read-back with the current step's compute."""
        for _ in nb.run_pipeline_stream(((n_pin, m_pin) for _ in range(k)), intr, theta,
                                        settings, device=dev):
            pass  # each step's log-depth is already in pinned host memory

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(fn, k, record):
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(k):
            res = fn()
            record(res)
        ev1.record()
        torch.cuda.synchronize()
        barrier()
        ms = ev0.elapsed_time(ev1) / k
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    fills = []
    iters = []

    def rec(res):
        fills.append(res[0].fill_report)
        iters.append(max(r.iterations for r in res))

    launches0 = _lib.launch_count()
    with ClockSampler(local_rank) as clk:
        ms = timed(step_device, args.steps, rec)
    launches = _lib.launch_count() - launches0
    clocks = clk.summary()

    # e2e through host buffers
    run_e2e(3)  # warms the pinned-host and device caching allocators
    torch.cuda.synchronize()
    e2e_steps = max(2, min(args.steps, 5))
    e2e_ms = timed(lambda: run_e2e(e2e_steps), 1, lambda r: None) / e2e_steps

    from paper_2510_11508_b200.shard import aggregate
    valid_total, _ = aggregate(valid_local, ms, dev)

    # roofline of the dominant kernel
    cg_ms = float(np.mean([f["cg_ms"] for f in fills]))
    px_iters = float(np.mean([f["px_iters"] for f in fills]))
    alg_bytes = BYTES_PER_PX_ITER * px_iters
    achieved = alg_bytes / (cg_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    prof = traffic_from_profile()
    roofline = {
        "kernel": "fill_cg_kernel (persistent batched CG, one launch per step)",
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4), "peak_source": peak_src,
        "traffic": (round(prof["dram_bytes_per_px_iter"] * px_iters) if prof else None),
        "traffic_note": ((prof["source"] + "; " + prof["note"]) if prof else
                         "no ncu capture committed"),
        "alg_bytes_per_launch": alg_bytes, "bytes_per_px_iter": BYTES_PER_PX_ITER,
        "survey_units": {
            "bytes_per_px_iter": SURVEY_BYTES_PER_PX_ITER,
            "achieved": round(SURVEY_BYTES_PER_PX_ITER * px_iters / (cg_ms * 1e-3) / 1e9, 1),
            "peak": SURVEY_PEAK_GBS,
            "note": "px-iterations/s x the SURVEY 8(d) two-sweep figure (72 B at 8-conn); the "
                    "single-sweep CG moves 37 B per px-iteration, so this exceeds what a "
                    "two-sweep PCG could reach at the same HBM traffic"},
        "px_iters_per_launch": px_iters, "kernel_ms": round(cg_ms, 3),
        "kernel_share_of_step": round(cg_ms / ms, 4),
        "fill_grid_ctas": fills[0]["grid"], "max_cg_iters": fills[0]["max_iters"],
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(normals_h[0], masks_h[0], intr_t[0], merge_freq)

    if rank == 0:
        h2d = int(n_pin.numel() * n_pin.element_size() + m_pin.numel() * m_pin.element_size())
        d2h = int(B * normals_h.shape[1] * normals_h.shape[2] * 8)  # float64 log-depth per map
        line = {
            "metric": "valid pixels/s end-to-end (component normal integration, run_pipeline)",
            "value": round(valid_total / (ms * 1e-3), 1),
            "unit": "valid_px/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 3),
            "higher_is_better": True,
            "scaling": "strong" if args.config == "C5" else "replicas",
            "vs_baseline": None,
            "dtype": "f32 CG vectors / f64 coefficients, dots, scales",
            "data": "synthetic (seeded generators, paper_2510_11508_b200/scenes.py)",
            "config": {
                "workload": desc,
                "maps_total": total_maps,
                "maps_per_rank": B,
                "valid_px_total": valid_total,
                "theta_c_deg": THETA_DEG,
                "connectivity": 8,
                "model": "milano",
                "reweighting": "soft",
                "merge_freq": merge_freq,
                "l2": "inputs larger than L2 (working set ~25 B/px x 67 M px)",
                "parallelism": f"maps sharded over {world} rank(s), no data-path collective",
            },
            "e2e": {"value": round(valid_total / (e2e_ms * 1e-3), 1), "unit": "valid_px/s",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "api": "run_pipeline_stream over pinned host batches: each step uploads its "
                           "normals + mask and reads every map's log-depth back; the next "
                           "step's upload and the previous step's read-back overlap the "
                           "current step's compute"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": round(launches / args.steps, 1),
            "outer_iterations_max": int(max(iters)),
        }
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- CPU legs


def _oracle_one(payload):
    normals, mask, intr, merge_freq = payload
    from oracle import normint_oracle as O
    t = time.perf_counter()
    O.run_pipeline(normals.astype(np.float64), mask, intr, float(np.deg2rad(THETA_DEG)),
                   O.Settings(freq_merging=merge_freq))
    return time.perf_counter() - t, int(mask.sum())


def cpu_baseline(normals, mask, intr, merge_freq):
    dt, valid = _oracle_one((normals, mask, intr, merge_freq))
    return {"value": round(valid / dt, 1), "unit": "valid_px/s", "cores": 1, "kind": "port",
            "sample": f"1 map ({mask.shape[1]}x{mask.shape[0]}, {valid} valid px) of the workload, "
                      f"oracle/normint_oracle.py run_pipeline, {dt:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import concurrent.futures as cf
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    procs = max(1, min(ncpu, args.maps if args.config == "C5" else 1))
    if args.config == "C5":
        payloads = [(*_gen_c5(i), None) for i in range(procs)]
    else:
        n, m, i, mf = _gen_cfg(args.config)
        payloads = [(n, m, i, mf)]
    warm = min(args.warmup, 1)
    times = []
    # one single-threaded process per core: pin every BLAS / OpenMP pool
    # before the workers start (they are spawned, so they inherit this env)
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS",
                "NUMEXPR_NUM_THREADS"):
        os.environ[var] = "1"
    import multiprocessing as mp
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn")) as ex:
        for s in range(warm + args.steps):
            t = time.perf_counter()
            out = list(ex.map(_oracle_one, payloads))
            dt = time.perf_counter() - t
            if s >= warm:
                times.append(dt)
    valid = sum(v for _, v in out)
    ms = 1e3 * float(np.mean(times))
    value = valid / (ms * 1e-3)
    line = {
        "impl": "reference",
        "metric": "valid pixels/s end-to-end (component normal integration, run_pipeline)",
        "value": round(value, 1), "unit": "valid_px/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": round(ms, 1), "higher_is_better": True,
        "scaling": "strong" if args.config == "C5" else "replicas", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generators, paper_2510_11508_b200/scenes.py)",
        "config": {"workload": make_desc(args), "maps_per_step": procs},
        "cpu_baseline": {"value": round(value, 1), "unit": "valid_px/s", "cores": procs,
                         "kind": "port",
                         "sample": f"{procs} map(s) per step, one process per core "
                                   f"(oracle/normint_oracle.py; the reference is pure Python and "
                                   f"cannot be installed on the GPU box)"},
        "e2e": {"value": round(value, 1), "unit": "valid_px/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_desc(args):
    if args.config == "C5":
        return f"C5: {args.maps} x 1024x1024 orthographic maps (seeds 100..{99 + args.maps}), 16 Voronoi cells"
    return args.config


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C5", choices=("C1", "C2", "C3", "C4", "C5"))
    ap.add_argument("--maps", type=int, default=64, help="C5 batch size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Benchmark: valid pixels/s of the component normal-integration hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
                    [--scaling weak|strong]

A step is one pass of the hot path (``run_pipeline`` semantics: normalise ->
components -> coefficients -> batched fill -> relative-scale loop with
merges -> gauge) over one batch of synthetic normal maps.  The default
workload is BASELINE.json config 5: a batch of 64 independent 1024x1024
orthographic maps (16 Voronoi cells).  Maps are independent objects, so with
N ranks every rank runs its own 64-map batch (weak scaling, rank r: seeds
100 + 64 r + i); ``--scaling strong`` splits one 64-map batch across the
ranks instead.

* ``value``: valid px/s with the normals already resident in HBM; whole-job
  = all ranks' valid pixels / max-over-ranks device time of a step.
* ``e2e``: the same through the public API from pinned HOST normals, with
  the host->device copy of the normals+mask and the device->host copy of the
  log-depth inside the timed region.
* ``roofline``: the dominant kernel, fine pass A of the multigrid fill:
  algorithmic bytes (58 B x active unit pixels per V-cycle, summed over the
  timed steps) over its CUDA-event time.
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

# Algorithmic HBM bytes per active unit pixel per V-cycle of the two fine
# passes of the multigrid-preconditioned CG (8-connectivity):
#  pass A reads r, s, w, dinv, hw, u, p, x (8 x f32), slot (u16), par0 (i32),
#         imask (u8) = 39 B, writes p, x, r', s' = 16 B, and the level-1
#         restriction b1, x1 (2 x f32 per 2x2 block) + its dinv1 read = 3 B;
#  pass B reads r, dinv, hw, par0 (4 x 4 B), imask, slot = 19 B and the
#         level-1 correction e1 (1 B), writes u, w = 8 B.
PASS_A_BYTES = 58
PASS_B_BYTES = 28
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


def map_indices(scaling, rank, world, nmaps):
    """C5 maps of a rank: weak scaling gives every rank its own batch of nmaps
    (config5_map indices 64 r .. 64 r + nmaps - 1, i.e. seeds 100 + 64 r + i);
    strong scaling splits one batch of nmaps into contiguous blocks."""
    if scaling == "weak":
        return list(range(rank * nmaps, (rank + 1) * nmaps))
    from paper_2510_11508_b200.shard import map_range
    lo, hi = map_range(rank, world, nmaps)
    return list(range(lo, hi))


def make_workload(config, rank, world, nmaps, scaling="weak"):
    """Return (normals (B,H,W,3) f32, masks (B,H,W) bool, intrinsics list,
    merge_freq, description, total maps)."""
    if config == "C5":
        idx = map_indices(scaling, rank, world, nmaps)
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
        total = nmaps * world if scaling == "weak" else nmaps
        return normals, masks, intr, None, None, total
    n, m, i, mf = _gen_cfg(config)
    return n[None], m[None], [i], mf, f"{config} (paper_2510_11508_b200/scenes.py)", 1


# -------------------------------------------------------------------- clocks


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    (nvidia_ml_py) every 50 ms when it loads, else nvidia-smi every 200 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, sm_max_mhz, [reason names])
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        visible = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.index
        if visible:  # CUDA's device numbering follows CUDA_VISIBLE_DEVICES, NVML's does not
            ids = [v.strip() for v in visible.split(",") if v.strip()]
            if self.index < len(ids) and ids[self.index].isdigit():
                idx = int(ids[self.index])
        h = nv.nvmlDeviceGetHandleByIndex(idx)
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        masks = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                              nv.nvmlDeviceGetCurrentClocksThrottleReasons)

        def sample():
            sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            bits = int(get_reasons(h))
            return sm, mx, [k for k, m in masks.items() if bits & m]

        sample()
        return sample

    def _smi(self):
        out = subprocess.run(
            ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
             "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode != 0 or not out.stdout.strip():
            return None
        r = [x.strip() for x in out.stdout.strip().split(",")]
        if not r[0].replace(".", "").isdigit() or not r[1].replace(".", "").isdigit():
            return None
        return float(r[0]), float(r[1]), [self.NAMES[k] for k in range(4)
                                           if len(r) > 4 + k and r[4 + k].lower() == "active"]

    def _run(self):
        sample, period = None, 0.2
        try:
            sample, period = self._nvml(), 0.05
            self.source = "nvml"
        except Exception:
            sample = None
        while not self._stop.is_set():
            try:
                row = sample() if sample else self._smi()
                if row:
                    self.rows.append(row)
            except Exception:
                pass
            self._stop.wait(period)

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
        reasons = sorted({k for r in self.rows for k in r[2]})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": self.source}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profile():
    """DRAM bytes per pixel of the fine passes from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "mg_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def mg_roofline(fills, step_ms):
    """Roofline of the multigrid fill's dominant fine pass: algorithmic bytes
    (PASS_*_BYTES x active unit pixels, summed over the V-cycles of every
    timed step) over its CUDA-event time on the fill's stream."""
    prof = [f["mg_profile"] for f in fills]
    pxv = float(np.mean([p["px_vcycles"] for p in prof]))
    vcyc = float(np.mean([f["mg"]["vcycles"] for f in fills]))
    t = {k: float(np.mean([p[k] for p in prof]))
         for k in ("pass_a_ms", "pass_b_ms", "coarse_ms", "scalar_ms")}
    peak, peak_src = measured_peak()
    passes = {}
    for name, key, nbytes in (("pass_a2_kernel<8>", "pass_a_ms", PASS_A_BYTES),
                              ("pass_b_kernel<8>", "pass_b_ms", PASS_B_BYTES)):
        ms_k = t[key]
        ach = nbytes * pxv / (ms_k * 1e-3) / 1e9 if ms_k > 0 else 0.0
        passes[name] = {"ms_per_step": round(ms_k, 3), "bytes_per_px_vcycle": nbytes,
                        "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 4)}
    top = max(passes, key=lambda k: passes[k]["ms_per_step"])
    nbytes = passes[top]["bytes_per_px_vcycle"]
    launches = max(vcyc, 1.0)
    prof_traffic = traffic_from_profile()
    traffic = None
    if prof_traffic and top in prof_traffic:
        traffic = round(prof_traffic[top]["dram_bytes_per_px"] * pxv / launches)
    fine_ms = t["pass_a_ms"] + t["pass_b_ms"]
    fine_ach = (PASS_A_BYTES + PASS_B_BYTES) * pxv / (fine_ms * 1e-3) / 1e9 if fine_ms else 0.0
    return {
        "kernel": top + " (fine pass of the multigrid-preconditioned CG fill)",
        "bound": "hbm", "achieved": passes[top]["achieved_gbs"], "peak": peak, "unit": "GB/s",
        "frac": passes[top]["frac"], "peak_source": peak_src,
        "traffic": traffic,
        "traffic_note": (prof_traffic["source"] if prof_traffic else "no ncu capture committed"),
        "alg_bytes_per_launch": round(nbytes * pxv / launches),
        "bytes_per_px_vcycle": nbytes,
        "px_vcycles_per_step": pxv, "vcycles_per_step": vcyc,
        "kernel_ms_per_launch": round(passes[top]["ms_per_step"] / launches, 4),
        "kernel_share_of_step": round(passes[top]["ms_per_step"] / step_ms, 4),
        "passes": passes,
        "fine_passes": {"achieved_gbs": round(fine_ach, 1), "frac": round(fine_ach / peak, 4),
                        "frac_vs_8tbs": round(fine_ach / SURVEY_PEAK_GBS, 4),
                        "share_of_step": round(fine_ms / step_ms, 4)},
        "stage_ms_per_step": {k: round(v, 3) for k, v in t.items()},
    }


# ------------------------------------------------------------------ our arm


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2510_11508_b200 as nb
    from paper_2510_11508_b200 import _lib

    normals_h, masks_h, intr_t, merge_freq, desc, total_maps = make_workload(
        args.config, rank, world, args.maps, args.scaling)
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

    gaps = []  # host time between the stream's yields (diagnostic: where a slow run lost its time)

    def run_e2e(k):
        """k steps through the serving API: every step copies its pinned host
        inputs to the device and reads every map's log-depth back into pinned
        host memory; run_pipeline_stream overlaps the next step's upload and
        the previous step's read-back with the current step's compute."""
        gaps.clear()
        t = time.perf_counter()
        for _ in nb.run_pipeline_stream(((n_pin, m_pin) for _ in range(k)), intr, theta,
                                        settings, device=dev):
            # each step's log-depth is already in pinned host memory
            t2 = time.perf_counter()
            gaps.append(round(1e3 * (t2 - t), 1))
            t = t2

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
    # What a serving process does after start-up: move the interpreter's
    # long-lived objects (torch, numpy, the generated scenes) out of the
    # collector's reach, so a full collection inside a step walks only that
    # step's records instead of pausing the host thread for ~35 ms.
    import gc
    gc.collect()
    gc.freeze()

    fills = []
    iters = []

    def rec(res):
        fills.append(res[0].fill_report)
        iters.append(max(r.iterations for r in res))

    _lib.set_fill_profiling(True)
    launches0 = _lib.launch_count()
    with ClockSampler(local_rank) as clk:
        ms = timed(step_device, args.steps, rec)
    launches = _lib.launch_count() - launches0
    _lib.set_fill_profiling(False)
    clocks = clk.summary()

    # e2e through host buffers
    run_e2e(3)  # warms the pinned-host and device caching allocators
    torch.cuda.synchronize()
    e2e_steps = max(2, min(2 * args.steps, 20))  # a serving stream: its two ends amortised
    from paper_2510_11508_b200 import pipeline as _pl
    allocs0 = torch.cuda.memory_stats(dev).get("num_device_alloc", 0)
    _pl._PIN_ALLOC_MS.clear()
    e2e_ms = timed(lambda: run_e2e(e2e_steps), 1, lambda r: None) / e2e_steps
    e2e_diag = {"device_allocs": int(torch.cuda.memory_stats(dev).get("num_device_alloc", 0)
                                     - allocs0),
                "pinned_alloc_ms_max": round(max(_pl._PIN_ALLOC_MS or [0.0]), 2)}

    from paper_2510_11508_b200.shard import gather_stats, whole_job
    stats = gather_stats(valid_local, ms, max(iters), B, dev)
    valid_total, ms = whole_job(stats)

    # roofline of the dominant kernel: the fine passes of the multigrid fill
    roofline = mg_roofline(fills, ms)
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
            "scaling": args.scaling if args.config == "C5" else "replicas",
            "vs_baseline": None,
            "dtype": "f32 CG vectors / f64 coefficients, dots, scales",
            "data": "synthetic (seeded generators, paper_2510_11508_b200/scenes.py)",
            "config": {
                **workload_config(args, world, merge_freq),
                "host": "gc.freeze() after the warm-up steps",
                "maps_per_rank": B,
                "valid_px_total": valid_total,
                "per_rank": [{"maps": int(r["maps"]), "valid_px": int(r["valid_px"]),
                              "ms_per_step": round(r["ms"], 3),
                              "outer_iterations": int(r["outer_iters"])} for r in stats],
            },
            "e2e": {"value": round(valid_total / (e2e_ms * 1e-3), 1), "unit": "valid_px/s",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps, "yield_gaps_ms": list(gaps), **e2e_diag,
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


def _oracle_c5(index):
    """One C5 map through the oracle port; the map is generated first, only
    the pipeline is timed."""
    return _oracle_one((*_gen_c5(index), None))


def run_reference(args, rank, world):
    if rank != 0:
        return
    import concurrent.futures as cf
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    procs = max(1, min(ncpu, args.maps if args.config == "C5" else 1))
    warm = args.warmup
    # one single-threaded process per core: pin every BLAS / OpenMP pool
    # before the workers start (they are spawned, so they inherit this env)
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS",
                "NUMEXPR_NUM_THREADS"):
        os.environ[var] = "1"
    import multiprocessing as mp
    times, valids = [], []
    # A step is bounded below by one map on one core (~12-24 s), so the run
    # cannot be made short by sampling less; what can give is the warm-up (a
    # numpy pipeline has nothing to warm): after the first step the remaining
    # warm-up steps are dropped if the projected run would exceed the budget,
    # and the line reports the warm-up actually executed.
    budget_s = float(os.environ.get("NI_REF_BUDGET_S", "540"))
    t_run = time.perf_counter()
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn")) as ex:
        s = 0
        executed_warm = 0
        while len(times) < args.steps:
            timed = executed_warm >= warm
            if args.config == "C5":
                # step s takes the next `procs` maps of the batch, so the
                # timed steps sweep the whole 64-map workload in turn
                idx = [(s * procs + k) % args.maps for k in range(procs)]
                out = list(ex.map(_oracle_c5, idx))
            else:
                n, m, i, mf = _gen_cfg(args.config)
                out = list(ex.map(_oracle_one, [(n, m, i, mf)]))
            s += 1
            if timed:
                times.append(max(dt for dt, _ in out))  # the processes run side by side
                valids.append(sum(v for _, v in out))
            else:
                executed_warm += 1
                per_step = (time.perf_counter() - t_run) / executed_warm
                if (executed_warm + 1 + args.steps) * per_step > budget_s:
                    warm = executed_warm  # no room for another warm-up step
    ms = 1e3 * float(np.mean(times))
    value = float(np.sum(valids)) / float(np.sum(times))
    line = {
        "impl": "reference",
        "metric": "valid pixels/s end-to-end (component normal integration, run_pipeline)",
        "value": round(value, 1), "unit": "valid_px/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "warmup_requested": args.warmup, "ms_per_step": round(ms, 1),
        "higher_is_better": True,
        "scaling": args.scaling if args.config == "C5" else "replicas", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generators, paper_2510_11508_b200/scenes.py)",
        "config": workload_config(args, world, None if args.config == "C5" else
                                  _gen_cfg(args.config)[3]),
        "cpu_baseline": {"value": round(value, 1), "unit": "valid_px/s", "cores": procs,
                         "kind": "port",
                         "sample": f"{procs} map(s) per step, one process per core "
                                   f"(oracle/normint_oracle.py; the reference is pure Python and "
                                   f"cannot be installed on the GPU box); step s runs maps "
                                   f"s*{procs} .. s*{procs}+{procs - 1} (mod {args.maps}), so the "
                                   f"warm-up + timed steps sweep the batch"},
        "e2e": {"value": round(value, 1), "unit": "valid_px/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(nproc: int) -> int:
    """`bench.py --gpus N` started without a launcher: re-run this command
    under torch.distributed.run, one rank per GPU on this node."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank, world):
    """The multi-rank plumbing of run_ours without a GPU: map split, one gloo
    process group, the stats all_gather and the whole-job aggregate."""
    import torch.distributed as dist

    from paper_2510_11508_b200.shard import gather_stats, map_range, whole_job
    if world > 1:
        dist.init_process_group("gloo")
    try:
        idx = map_indices(args.scaling, rank, world, args.maps)
        t = time.perf_counter()
        valid = 0
        for i in idx:
            _, m, _ = _gen_c5(i)
            valid += int(m.sum())
        ms = 1e3 * (time.perf_counter() - t)
        stats = gather_stats(valid, ms, 1, len(idx))
        valid_total, ms_max = whole_job(stats)
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "value": valid_total / ms_max * 1e3,
                              "scaling": args.scaling,
                              "config": {"maps_total": sum(int(r["maps"]) for r in stats),
                                         "valid_px_total": valid_total,
                                         "per_rank": [{"maps": int(r["maps"]),
                                                       "valid_px": int(r["valid_px"])}
                                                      for r in stats]}}), flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()


def workload_config(args, world, merge_freq):
    """The config keys both arms report for the same workload."""
    return {
        "workload": make_desc(args),
        "maps_total": (args.maps * (world if args.scaling == "weak" else 1)
                       if args.config == "C5" else 1),
        "theta_c_deg": THETA_DEG,
        "connectivity": 8,
        "model": "milano",
        "reweighting": "soft",
        "merge_freq": merge_freq,
        "l2": ("inputs larger than L2 (working set ~25 B/px x 67 M px)" if args.config == "C5"
               else "single-map config (a parity/latency line, not the bench workload)"),
        "parallelism": (f"{world} rank(s), each its own batch of {args.maps} maps (weak scaling), "
                        "no data-path collective" if args.scaling == "weak" and args.config == "C5"
                        else f"maps sharded over {world} rank(s), no data-path collective"),
    }


def make_desc(args):
    if args.config == "C5":
        return (f"C5: {args.maps} x 1024x1024 orthographic maps per rank (BASELINE config 5; "
                f"rank r: seeds 100 + {args.maps} r .. + {args.maps - 1}), 16 Voronoi cells"
                if args.scaling == "weak" else
                f"C5: {args.maps} x 1024x1024 orthographic maps (seeds 100..{99 + args.maps}) "
                "split across the ranks, 16 Voronoi cells")
    return f"{args.config} (paper_2510_11508_b200/scenes.py)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C5", choices=("C1", "C2", "C3", "C4", "C5"))
    ap.add_argument("--maps", type=int, default=64, help="C5 batch size (per rank when weak)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: every rank its own 64-map batch (independent maps, SURVEY 8(e)); "
                         "strong: one 64-map batch split across the ranks")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / gather plumbing only: gloo, no GPU work (CPU tests)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.dry_run:
        dry_run(args, rank, world)
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

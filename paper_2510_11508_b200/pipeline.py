"""Drop-in ``run_pipeline`` (pipeline.py:105-248) on the B200 kernels.

The host code keeps the reference's signature, options, diagnostics records
and result type; every data-parallel step runs in ``libnormint_b200.so``
through the C ABI.  The host only makes the scalar decisions of Algorithm 1
(energy convergence test, merge schedule), reading back a few bytes per
outer iteration.

``run_pipeline_batch`` runs B independent maps of one size as a single grid
(one components launch, one coefficients launch, ONE batched fill over the
components of all maps), then the small per-map outer loops.
"""

from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import functools
import hashlib
import math
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, devmem
from .errors import EmptyMask
from .geometry import (CameraIntrinsics, LogDepthMap, NormalMap, _device, _stream, as_intrinsics,
                       as_normal_map)
from .settings import CONTINUITY_MODELS, SolveSettings, WeightParams, as_settings, as_weights

ENERGY_FLOOR = 1e-300  # pipeline.py:55
# fill solver: "mg" (multigrid-preconditioned CG, default) or "cg" (the
# round-1 unpreconditioned single-sweep CG kernel; experiments only)
_FILL_SOLVER = os.environ.get("NI_FILL_SOLVER", "mg")


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _ws(nbytes: int, dev) -> torch.Tensor:
    return devmem.empty(max(int(nbytes), 1), torch.uint8, dev)


def _ms(start: float) -> float:
    return (time.perf_counter() - start) * 1e3


# ----------------------------------------------------------------- threshold


def _f64_key(x: float) -> int:
    bits = int(np.array([x], np.float64).view(np.int64)[0])
    return bits if bits >= 0 else -(bits & 0x7FFFFFFFFFFFFFFF)


def _f64_from_key(k: int) -> float:
    bits = k if k >= 0 else ((-k) | (1 << 63)) - (1 << 64)
    return float(np.array([bits], np.int64).view(np.float64)[0])


def dot_cutoff(theta_c: float) -> float:
    """Smallest float64 d with numpy.arccos(clip(d, -1, 1)) < theta_c (memoised:
    the bisection is ~0.35 ms of host time, a tenth of a small map's run)."""
    return _dot_cutoff(float(theta_c))


@functools.lru_cache(maxsize=64)
def _dot_cutoff(theta_c: float) -> float:
    """Smallest float64 d with numpy.arccos(clip(d, -1, 1)) < theta_c.

    The reference keeps an edge iff arccos(clip(n_a . n_b)) < theta_c
    (graph.py:92, 159).  numpy's arccos is monotone, so the kept set equals
    {dot >= d*}; d* is found by bisection over the float64 lattice with the
    host's own numpy arccos (evaluated through a full SIMD-width vector, the
    same inner loop the reference runs on its edge arrays).  The GPU then
    needs no transcendental at all and reproduces the kept set bit for bit.
    """
    theta_c = float(theta_c)

    def kept(d):
        v = np.clip(np.full(64, d, np.float64), -1.0, 1.0)
        return bool(np.arccos(v)[17] < theta_c)

    if not kept(1.0):
        return math.inf
    if kept(-1.0):
        return -math.inf
    lo, hi = _f64_key(-1.0), _f64_key(1.0)
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if kept(_f64_from_key(mid)):
            hi = mid
        else:
            lo = mid
    return _f64_from_key(hi)


# ------------------------------------------------------------------ results


class Partition:
    """Assignment of every valid pixel to a component (graph.py:101-130).

    ``labels`` (host, int64, -1 invalid) is materialised lazily from the
    device tensor ``labels_t`` (int32).  Labels are canonical.
    """

    def __init__(self, labels_t: torch.Tensor, component_count: int, version: int = 0,
                 label_base: int = 0):
        self.labels_t = labels_t
        self.component_count = int(component_count)
        self.version = int(version)
        self.label_base = int(label_base)
        self._labels = None

    @property
    def labels(self) -> np.ndarray:
        if self._labels is None:
            a = self.labels_t.to(torch.int64).cpu().numpy()
            if self.label_base:
                a = np.where(a >= 0, a - self.label_base, -1)
            a.flags.writeable = False
            self._labels = a
        return self._labels

    @property
    def sizes(self) -> np.ndarray:
        lab = self.labels
        return np.bincount(lab[lab >= 0], minlength=self.component_count)

    def pixels_of(self, c: int) -> np.ndarray:
        return np.flatnonzero(self.labels == c)


@dataclass
class PipelineResult:
    """Everything the component pipeline produced (pipeline.py:91-102)."""

    log_depth: LogDepthMap
    filled: LogDepthMap
    partition0: Partition
    partition: Partition
    records: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    iterations: int = 0
    energies: list = field(default_factory=list)
    fill_iterations: np.ndarray | None = None  # per component CG iterations (GPU extra)
    fill_report: dict | None = None  # device timing of the batched fill (GPU extra)


def _has_converged(e_t: float, e_prev: float, t: int, settings: SolveSettings) -> bool:
    """pipeline.py:66-83."""
    if t >= settings.max_iters:
        return True
    if e_t <= ENERGY_FLOOR:
        return True
    if t <= settings.alignment_iters + 1 or e_prev <= ENERGY_FLOOR:
        return False
    return abs(e_t - e_prev) / e_prev < settings.delta_e_max


def _digest(z_map: torch.Tensor) -> str:
    """First 16 hex digits of SHA-256 over the map's float64 z (pipeline.py:58-59)."""
    return hashlib.sha256(z_map.cpu().numpy().tobytes()).hexdigest()[:16]


def _digest_async(snap: torch.Tensor, ready: torch.cuda.Event) -> str:
    """_digest of a device snapshot, from a worker thread: the copy runs on a
    side stream into pinned memory (the pipeline's stream keeps going) and
    the hash reads the pinned buffer in place with the GIL released."""
    side = torch.cuda.Stream(device=snap.device)
    host = torch.empty(snap.numel(), dtype=torch.float64, pin_memory=True)
    with torch.cuda.stream(side):
        side.wait_event(ready)
        host.copy_(snap, non_blocking=True)
    side.synchronize()
    return hashlib.sha256(memoryview(host.numpy())).hexdigest()[:16]


# ------------------------------------------------------------------- engine


class _Grid:
    """Device state shared by every stage of one (batched) run."""

    def __init__(self, nmap: NormalMap, connectivity: int, model: str):
        self.nmap = nmap
        self.dev = nmap.device
        self.stream = _stream(self.dev)
        self.B, self.H, self.W = nmap.batch, nmap.height, nmap.width
        self.hw = self.H * self.W
        self.npix = nmap.npix
        self.conn = connectivity
        self.kf = 4 if connectivity == 8 else 2
        self.model = CONTINUITY_MODELS.index(model)
        self.lib = _lib.load()
        self.stats = torch.zeros(6, dtype=torch.int64, device=self.dev)

    def s(self):
        return C.c_void_p(self.stream)


def _components(g: _Grid, theta_c):
    lib = g.lib
    labels = devmem.empty(g.npix, torch.int32, g.dev)
    count = torch.zeros(1, dtype=torch.int32, device=g.dev)
    map_first = torch.zeros(g.B + 1, dtype=torch.int32, device=g.dev)
    ws = _ws(_lib.size_query(lib.ni_components_workspace_size, g.B, g.H, g.W), g.dev)
    cutoff = 0.0 if theta_c is None else dot_cutoff(theta_c)
    _lib.check(lib.ni_components(_ptr(g.nmap.n_soa), _ptr(g.nmap.valid_t), g.B, g.H, g.W, g.conn,
                                 C.c_double(cutoff), 1 if theta_c is None else 0, _ptr(labels),
                                 _ptr(count), _ptr(map_first), _ptr(g.stats), _ptr(ws), ws.numel(),
                                 g.s()), "form_components")
    return labels, map_first


def _coefficients(g: _Grid, intrinsics: list[CameraIntrinsics]):
    lib = g.lib
    intr = torch.tensor([i.as_tuple() for i in intrinsics], dtype=torch.float64).to(g.dev)
    omega_a = devmem.empty((g.kf, g.npix), torch.float64, g.dev)
    omega_b = devmem.empty((g.kf, g.npix), torch.float64, g.dev) if g.model == 1 else None
    gamma = devmem.empty(g.npix, torch.float64, g.dev)
    eflags = devmem.empty(g.npix, torch.uint8, g.dev)
    g.map_counts = torch.zeros(2 * g.B, dtype=torch.int64, device=g.dev)
    _lib.check(lib.ni_coefficients(_ptr(g.nmap.n_soa), _ptr(g.nmap.valid_t), _ptr(intr), g.B, g.H,
                                   g.W, g.conn, g.model, _ptr(omega_a), _ptr(omega_b), _ptr(gamma),
                                   _ptr(eflags), _ptr(g.stats), _ptr(g.map_counts), g.s()),
               "build_edge_coefficients")
    return omega_a, omega_b, gamma, eflags


# weight modes of ni_edge_weights (ni_edges.cuh)
EW_UNIFORM, EW_BILATERAL, EW_FULL = 0, 1, 2


def _edge_weights(g: _Grid, co, z: torch.Tensor, wmode: int, weights: WeightParams):
    """Directed weights of every forward pixel edge at state z (continuity.py:292-331,
    solver.py:253-278)."""
    omega_a, omega_b, gamma, eflags = co
    w_a = devmem.empty((g.kf, g.npix), torch.float64, g.dev)
    w_b = devmem.empty((g.kf, g.npix), torch.float64, g.dev)
    _lib.check(g.lib.ni_edge_weights(_ptr(z), _ptr(omega_a), _ptr(omega_b), _ptr(gamma),
                                     _ptr(eflags), g.B, g.H, g.W, g.conn, g.model, wmode,
                                     weights.mode_code, C.c_double(weights.k),
                                     C.c_double(weights.outlier_low),
                                     C.c_double(weights.outlier_high), _ptr(w_a), _ptr(w_b),
                                     g.s()), "edge_weights")
    return w_a, w_b


def _pair_energy(g: _Grid, co, x: torch.Tensor, wts) -> torch.Tensor:
    """Per-map energy of the pixel pair system at x (pipeline.py:336-337)."""
    omega_a, omega_b, _, eflags = co
    out = devmem.empty(g.B, torch.float64, g.dev)
    ws = _ws(_lib.size_query(g.lib.ni_pair_energy_workspace_size, g.B), g.dev)
    _lib.check(g.lib.ni_pair_energy(_ptr(x), _ptr(omega_a), _ptr(omega_b), _ptr(wts[0]),
                                    _ptr(wts[1]), _ptr(eflags), g.B, g.H, g.W, g.conn, g.model,
                                    _ptr(out), _ptr(ws), ws.numel(), g.s()), "pair_energy")
    return out


def _fill_mg_buffers(g: _Grid, count: int):
    """Output and workspace buffers of ni_fill_mg.  run_pipeline_batch makes
    them while the coefficients kernel still runs (before its first host
    read-back), so the allocations are off the GPU's critical path."""
    z = devmem.empty(g.npix, torch.float64, g.dev)
    iters = torch.zeros(max(count, 1), dtype=torch.int32, device=g.dev)
    status = torch.zeros(max(count, 1), dtype=torch.int32, device=g.dev)
    nbytes = _lib.size_query(g.lib.ni_fill_mg_workspace_size, g.B, g.H, g.W, g.conn, count)
    return z, iters, status, nbytes, _ws(nbytes, g.dev)


def _fill_mg(g: _Grid, labels, count, co, settings: SolveSettings):
    """The fill at z = 0 (solver.py:195-239) as one batched multigrid-
    preconditioned CG over every solve unit of the batch (ni_fill_mg)."""
    lib = g.lib
    omega_a, omega_b, gamma, eflags = co
    pre = getattr(g, "fill_buffers", None)
    g.fill_buffers = None
    z, iters, status, nbytes, ws0 = pre if pre is not None else _fill_mg_buffers(g, count)
    for attempt in range(3):  # the hierarchy's size depends on the data: retry with what it needs
        ws = ws0 if attempt == 0 else _ws(nbytes, g.dev)
        ws0 = None
        need = C.c_size_t(0)
        st = lib.ni_fill_mg(_ptr(labels), count, _ptr(omega_a), _ptr(omega_b), _ptr(gamma),
                            _ptr(eflags), g.B, g.H, g.W, g.conn, g.model,
                            C.c_double(settings.cg_tol), int(settings.cg_max_iters), _ptr(z),
                            _ptr(iters), _ptr(status), _ptr(ws), ws.numel(), C.byref(need),
                            g.s())
        if st != _lib.NI_ERR_WORKSPACE:
            break
        del ws
        nbytes = max(int(need.value), nbytes + 1)
    _lib.check(st, "fill_components")
    return z, iters[:count], status[:count]


def _fill(g: _Grid, labels, count, co, settings: SolveSettings, wts=None):
    """Batched per-component CG (solver.py:195-239); ``wts`` = per-edge weights
    (w_a, w_b) for the refill pass / the pixel baseline, None for the fill
    (which runs the multigrid-preconditioned solve unless NI_FILL_SOLVER=cg)."""
    if wts is None and _FILL_SOLVER != "cg":
        return _fill_mg(g, labels, count, co, settings)
    lib = g.lib
    omega_a, omega_b, gamma, eflags = co
    z = devmem.empty(g.npix, torch.float64, g.dev)
    iters = torch.zeros(max(count, 1), dtype=torch.int32, device=g.dev)
    status = torch.zeros(max(count, 1), dtype=torch.int32, device=g.dev)
    ws = _ws(_lib.size_query(lib.ni_fill_workspace_size, g.B, g.H, g.W, g.conn, count,
                             int(wts is not None)), g.dev)
    w_a, w_b = (None, None) if wts is None else wts
    _lib.check(lib.ni_fill(_ptr(labels), count, _ptr(omega_a), _ptr(omega_b), _ptr(gamma),
                           _ptr(eflags), _ptr(w_a), _ptr(w_b), g.B, g.H, g.W, g.conn, g.model,
                           C.c_double(settings.cg_tol), int(settings.cg_max_iters), _ptr(z),
                           _ptr(iters), _ptr(status), _ptr(ws), ws.numel(), g.s()),
               "fill_components")
    return z, iters[:count], status[:count]


class _BatchLoop:
    """The outer relative-scale loops of all maps of a batch in lockstep
    (pipeline.py:169-227): the maps step together through one batched call
    per stage, each keeping its own CG, energy, merges and convergence test;
    a map leaves the loop once it has converged.  Component ids are the
    batch's global labels (map m owns [first[m], first[m] + count[m]))."""

    def __init__(self, g: _Grid, labels: torch.Tensor, first: np.ndarray, counts, co,
                 settings: SolveSettings, weights: WeightParams):
        self.g, self.labels = g, labels
        self.first = np.ascontiguousarray(first, dtype=np.int32)  # [B+1], fixed
        self.count = np.ascontiguousarray(counts, dtype=np.int32)  # [B], shrinks with merges
        self.C = max(int(self.first[-1]), 1)  # component id space
        self.co = co
        self.settings, self.weights = settings, weights
        self.keys = None
        self.K = 0
        self.quot = None
        self.map_edges = np.zeros(g.B, dtype=np.int32)
        dev = g.dev
        self.energy = torch.zeros(g.B, dtype=torch.float64, device=dev)
        self.ok = torch.zeros(g.B, dtype=torch.int32, device=dev)
        self.merge_energy = torch.zeros(g.B, dtype=torch.float64, device=dev)
        self.new_count = torch.zeros(g.B, dtype=torch.int32, device=dev)
        # deferred scales: the loop's state is z + zshift[label]; folded into
        # z (ni_apply_shift) before a merge relabels a map and at the end
        self.zshift = None
        self._mapws = devmem.empty(4 * g.B, torch.uint8, dev)
        self._fused_bufs = None

    def defer_scales(self):
        self.zshift = torch.zeros(self.C, dtype=torch.float64, device=self.g.dev)

    def fold_scales(self, z: torch.Tensor, maps: np.ndarray):
        if self.zshift is None or len(maps) == 0:
            return
        g = self.g
        mp = np.ascontiguousarray(maps, dtype=np.int32)
        _lib.check(g.lib.ni_apply_shift(_ptr(z), _ptr(self.zshift), _ptr(self.labels), g.B, g.H,
                                        g.W, self._hp(mp), len(mp), _ptr(self._mapws),
                                        self._mapws.numel(), g.s()), "apply_scales")

    @staticmethod
    def _hp(a: np.ndarray) -> C.c_void_p:
        return C.c_void_p(a.ctypes.data)

    def initial_keys(self):
        g, lib = self.g, self.g.lib
        out = devmem.empty(g.npix * g.kf, torch.int32, g.dev)
        n = torch.zeros(1, dtype=torch.int32, device=g.dev)
        ws = _ws(_lib.size_query(lib.ni_inter_edges_workspace_size, g.B, g.H, g.W, g.conn), g.dev)
        _lib.check(lib.ni_inter_edges(_ptr(self.labels), _ptr(self.co[3]), g.B, g.H, g.W, g.conn,
                                      _ptr(out), _ptr(n), _ptr(ws), ws.numel(), g.s()),
                   "build_quotient")
        self.K = int(n.item())
        self.keys = out[:self.K].clone()

    def filter_keys(self, keep: np.ndarray):
        """Drop edges of maps that left the loop and edges a merge made intra."""
        g, lib = self.g, self.g.lib
        mk = torch.from_numpy(keep.astype(np.uint8)).to(g.dev)
        out = devmem.empty(max(self.K, 1), torch.int32, g.dev)
        n = torch.zeros(1, dtype=torch.int32, device=g.dev)
        ws = _ws(_lib.size_query(lib.ni_keys_filter_workspace_size, self.K), g.dev)
        _lib.check(lib.ni_keys_filter(_ptr(self.keys), self.K, _ptr(self.labels), _ptr(mk), g.H,
                                      g.W, g.conn, _ptr(out), _ptr(n), _ptr(ws), ws.numel(), g.s()),
                   "build_quotient")
        self.K = int(n.item())
        self.keys = out[:self.K]

    def build(self):
        g, lib = self.g, self.g.lib
        qbytes = _lib.size_query(lib.ni_quotient_workspace_size, self.K, self.C, g.B)
        self.quot = _ws(qbytes, g.dev)
        npairs = C.c_int32(0)
        self.map_edges = np.zeros(g.B, dtype=np.int32)
        _lib.check(lib.ni_quotient_build(_ptr(self.keys), self.K, _ptr(self.labels), self.C, g.B,
                                         g.H, g.W, g.conn, _ptr(self.quot), self.quot.numel(),
                                         C.byref(npairs), self._hp(self.map_edges), g.s()),
                   "build_quotient")

    def step(self, z: torch.Tensor, t: int, active: np.ndarray, live: torch.Tensor | None = None):
        g, lib = self.g, self.g.lib
        st, wp = self.settings, self.weights
        omega_a, omega_b, gamma, eflags = self.co
        scales = devmem.empty(self.C, torch.float64, g.dev)
        residual = devmem.empty(max(2 * self.K, 1), torch.float64, g.dev)
        wts = devmem.empty(max(2 * self.K, 1), torch.float64, g.dev)
        ws = _ws(_lib.size_query(lib.ni_scale_step_workspace_size, self.K, self.C, g.B), g.dev)
        _lib.check(lib.ni_scale_step(
            _ptr(self.quot), self.quot.numel(), self.K, self.C, g.B, self._hp(self.first),
            self._hp(self.count), self._hp(active), len(active), _ptr(self.labels),
            _ptr(omega_a), _ptr(omega_b), _ptr(gamma), _ptr(eflags), g.H, g.W, g.conn, g.model, t,
            st.alignment_iters, wp.mode_code, C.c_double(wp.k), C.c_double(wp.outlier_low),
            C.c_double(wp.outlier_high), C.c_double(st.cg_tol), int(st.cg_max_iters), _ptr(z),
            _ptr(self.zshift), _ptr(live), _ptr(scales), _ptr(residual), _ptr(wts), _ptr(self.energy), _ptr(self.ok), _ptr(ws),
            ws.numel(), g.s()), "relative_scale_step")
        self.last_scales = scales
        return residual, wts

    def step_fused(self, z: torch.Tensor, t: int, k: int, maps: np.ndarray, dl: "_DeviceLoop"):
        """Iterations t .. t + k - 1 with the convergence test of the
        small-quotient maps ``maps``, a CTA per map, in one launch
        (ni_scale_step_fused)."""
        g, lib = self.g, self.g.lib
        st, wp = self.settings, self.weights
        omega_a, omega_b, gamma, eflags = self.co
        if self._fused_bufs is None or self._fused_bufs[0].numel() < self.C:
            self._fused_bufs = (devmem.empty(self.C, torch.float64, g.dev),
                                devmem.empty(max(2 * self.K, 1), torch.float64, g.dev),
                                devmem.empty(max(2 * self.K, 1), torch.float64, g.dev),
                                _ws(_lib.size_query(lib.ni_scale_step_workspace_size, self.K,
                                                    self.C, g.B), g.dev))
        scales, residual, wts, ws = self._fused_bufs
        mp = np.ascontiguousarray(maps, dtype=np.int32)
        _lib.check(lib.ni_scale_step_fused(
            _ptr(self.quot), self.quot.numel(), self.K, self.C, g.B, self._hp(self.first),
            self._hp(self.count), self._hp(mp), len(mp), _ptr(self.labels), _ptr(omega_a),
            _ptr(omega_b), _ptr(gamma), _ptr(eflags), g.H, g.W, g.conn, g.model, t, k,
            st.alignment_iters, wp.mode_code, C.c_double(wp.k), C.c_double(wp.outlier_low),
            C.c_double(wp.outlier_high), C.c_double(st.cg_tol), int(st.cg_max_iters), _ptr(z),
            _ptr(self.zshift), _ptr(scales), _ptr(residual), _ptr(wts), _ptr(self.energy),
            _ptr(self.ok), st.max_iters, C.c_double(st.delta_e_max), _ptr(dl.e_prev),
            _ptr(dl.live), _ptr(dl.iters), _ptr(dl.e_hist), _ptr(dl.ok_hist), dl.T,
            _ptr(dl.nlive), _ptr(ws), ws.numel(), g.s()), "relative_scale_step")

    def fusable(self, active: np.ndarray) -> np.ndarray:
        """Maps of ``active`` whose quotient fits one CTA (ni_scale_fused_limits)."""
        if self.K == 0 or self.zshift is None:
            return np.zeros(len(active), dtype=bool)
        me, mc = C.c_int32(0), C.c_int32(0)
        self.g.lib.ni_scale_fused_limits(C.byref(me), C.byref(mc))
        return ((self.map_edges[active] <= me.value) & (self.count[active] <= mc.value))

    def merge(self, residual, wts, merging: np.ndarray):
        g, lib = self.g, self.g.lib
        ws = _ws(_lib.size_query(lib.ni_merge_workspace_size, self.K, self.C, g.B), g.dev)
        _lib.check(lib.ni_merge(_ptr(self.quot), self.quot.numel(), self.K, self.C, g.B,
                                self._hp(self.first), self._hp(self.count), self._hp(merging),
                                len(merging), _ptr(self.labels), g.H, g.W, _ptr(residual),
                                _ptr(wts), _ptr(self.new_count), _ptr(self.merge_energy),
                                _ptr(ws), ws.numel(), g.s()), "merge_components")


class _DeviceLoop:
    """Chunks of outer iterations with the convergence test on the device
    (ni_loop_decide): maps that converge inside a chunk sit the remaining
    steps out (live flag 0); the host reads energies, cap flags and
    convergence points back once per chunk and writes the same records as the
    per-iteration loop.  A chunk never contains a merge step."""

    MAX_CHUNK = 64
    LAG = 3  # iterations enqueued ahead of the last one whose outcome the host has seen
    _host_cache: dict = {}

    def __init__(self, g: _Grid, settings: SolveSettings):
        self.g, self.settings = g, settings
        dev, B, T = g.dev, g.B, max(settings.max_iters, 1)
        self.T = T
        self.live = torch.zeros(B, dtype=torch.int32, device=dev)
        self.iters = torch.zeros(B, dtype=torch.int32, device=dev)
        self.e_hist = torch.zeros((B, T), dtype=torch.float64, device=dev)
        self.ok_hist = torch.zeros((B, T), dtype=torch.int32, device=dev)
        self.e_prev = torch.zeros(B, dtype=torch.float64, device=dev)
        self.nlive = torch.zeros(1, dtype=torch.int32, device=dev)
        # the pinned counters and the events are per device, made once (a pinned
        # allocation + 64 event creations cost ~0.5 ms of host time per run)
        key = (dev.index if dev.index is not None else torch.cuda.current_device(),
               threading.get_ident())
        if key not in _DeviceLoop._host_cache:
            _DeviceLoop._host_cache[key] = (
                torch.zeros(self.MAX_CHUNK, dtype=torch.int32, pin_memory=True),
                [torch.cuda.Event() for _ in range(self.MAX_CHUNK)])
        self.nlive_host, self.events = _DeviceLoop._host_cache[key]
        self.t0 = 0
        self.wall = 0.0

    def length(self, t: int) -> int:
        st = self.settings
        k = st.max_iters - t
        if st.freq_merging is not None:  # stop before the next step t' with (t' + 1) % f == 0
            k = min(k, (st.freq_merging - 1 - t) % st.freq_merging)
        return min(k, self.MAX_CHUNK)

    def run(self, loop: "_BatchLoop", z, t: int, k: int, active: np.ndarray) -> int:
        g, st = self.g, self.settings
        start = time.perf_counter()
        act = torch.from_numpy(np.ascontiguousarray(active, dtype=np.int32)).to(g.dev)
        self.live.zero_()
        self.live[act.long()] = 1
        self.iters.zero_()
        self.nlive.fill_(len(active))
        self.t0 = t
        stream = torch.cuda.current_stream(g.dev)
        fuse = loop.fusable(active)
        fused, rest = active[fuse], active[~fuse]
        if len(fused):  # their whole chunk in one launch
            loop.step_fused(z, t, k, fused, self)
        if not len(rest):
            self.wall = _ms(start) / k
            return t + k
        act = torch.from_numpy(np.ascontiguousarray(rest, dtype=np.int32)).to(g.dev)
        for i in range(k):
            # stop once every map has converged, judged LAG iterations behind
            # the queue head (at most LAG iterations run with no map left)
            if i >= self.LAG:
                self.events[i - self.LAG].synchronize()
                if int(self.nlive_host[i - self.LAG]) == 0:
                    break
            loop.step(z, t, rest, self.live)
            t += 1
            _lib.check(g.lib.ni_loop_decide(
                _ptr(loop.energy), _ptr(loop.ok), _ptr(act), len(rest), t, st.max_iters,
                st.alignment_iters, C.c_double(st.delta_e_max), _ptr(self.e_prev),
                _ptr(self.live), _ptr(self.iters), _ptr(self.e_hist), _ptr(self.ok_hist),
                self.T, _ptr(self.nlive), g.s()), "convergence test")
            self.nlive_host[i:i + 1].copy_(self.nlive, non_blocking=True)
            self.events[i].record(stream)
        self.wall = _ms(start) / max(t - self.t0, 1)
        return t

    def collect(self, loop, active, t, e_prev, energies, records, warnings, iters):
        """Read the chunk's outcome back.  Returns (still, finish): the maps still
        in the loop, and a callable that writes the chunk's records -- ~0.5 ms of
        host work for 64 maps x 37 iterations, which the caller runs after it has
        enqueued the GPU work that does not depend on it."""
        t0 = self.t0
        host = torch.cat([self.e_hist[:, t0:t].reshape(-1),
                          self.ok_hist[:, t0:t].reshape(-1).to(torch.float64),
                          self.live.to(torch.float64), self.iters.to(torch.float64),
                          self.e_prev]).cpu().numpy()
        B, k = self.g.B, t - t0
        eh = host[:B * k].reshape(B, k)
        oh = host[B * k:2 * B * k].reshape(B, k)
        live = host[2 * B * k:2 * B * k + B]
        conv = host[2 * B * k + B:2 * B * k + 2 * B]
        ep = host[2 * B * k + 2 * B:]
        still = []
        for m in active:
            m = int(m)
            e_prev[m] = float(ep[m])
            if live[m]:
                still.append(m)
            else:
                iters[m] = int(conv[m])
        wall, counts = self.wall, [int(c) for c in loop.count]

        def finish():
            for m in active:
                m = int(m)
                last = int(conv[m]) if not live[m] else t
                for tt in range(t0 + 1, last + 1):
                    e_t = float(eh[m, tt - 1 - t0])
                    if not oh[m, tt - 1 - t0]:
                        warnings[m].append(f"iteration {tt - 1}: cg hit iteration cap")
                    energies[m].append(e_t)
                    records[m].append({"t": tt, "E_t": e_t, "component_count": counts[m],
                                       "merge_performed": False, "wall_ms": wall})

        return still, finish

    def sync_prev(self, e_prev: np.ndarray):
        self.e_prev.copy_(torch.from_numpy(np.ascontiguousarray(e_prev, dtype=np.float64)))


def _validate(model, connectivity):
    if model not in CONTINUITY_MODELS:
        raise ValueError(f"unknown continuity model {model!r}")
    if connectivity not in (4, 8):
        raise ValueError("connectivity must be 4 or 8")
    if model == "bini" and connectivity == 8:
        raise ValueError(
            "the pinhole finite-difference model defines no diagonal "
            "coefficient; use connectivity=4 with model='bini'"
        )


def run_pipeline_batch(
    nmap: NormalMap,
    intrinsics,
    theta_c: float | None,
    settings: SolveSettings | None = None,
    weights: WeightParams | None = None,
    connectivity: int = 8,
    model: str = "milano",
    gauge_depth: float | None = None,
) -> list[PipelineResult]:
    """``run_pipeline`` over the B maps of a batched NormalMap.

    ``intrinsics`` is one CameraIntrinsics or a list of B.  Returns one
    PipelineResult per map, bit-identical in content to what
    ``run_pipeline`` returns for that map alone (every reduction of a map
    runs in an order that does not depend on the other maps;
    tests/test_gpu_edge_cases.py::test_batch_bit_identical_to_single_maps).
    """
    settings = as_settings(settings) or SolveSettings()
    weights = as_weights(weights) or WeightParams()
    _validate(model, connectivity)
    nmap = as_normal_map(nmap)
    B = nmap.batch
    intr = list(intrinsics) if isinstance(intrinsics, (list, tuple)) else [intrinsics] * B
    intr = [as_intrinsics(i) for i in intr]
    if len(intr) != B:
        raise ValueError("need one CameraIntrinsics per map")
    records = [[] for _ in range(B)]
    warnings = [[] for _ in range(B)]
    run_start = time.perf_counter()
    g = _Grid(nmap, connectivity, model)
    if nmap.valid_count == 0:
        raise EmptyMask("normal map has no valid pixel")

    t0 = time.perf_counter()
    labels, map_first = _components(g, theta_c)
    valid_sum = g.nmap.valid_t.view(B, -1).sum(dim=1, dtype=torch.int64)
    first = map_first.cpu().numpy().astype(np.int64)
    stats = g.stats.cpu().numpy()
    valid_per_map = valid_sum.cpu().numpy()
    comp_ms = _ms(t0)
    if B > 1 and (valid_per_map == 0).any():
        raise EmptyMask("normal map has no valid pixel")
    # The coefficients do not depend on the labels: their kernel is enqueued
    # before the host writes the records of the first stages, and its counters
    # are read back only after the fill (whose first read-back waits for it
    # anyway), so neither costs the GPU idle time.
    t0 = time.perf_counter()
    labels0 = labels.clone()
    co = _coefficients(g, intr)
    if _FILL_SOLVER != "cg" and not settings.refill_reweighted:
        g.fill_buffers = _fill_mg_buffers(g, int(first[B]))  # while the kernel runs
    coef_ms = _ms(t0)
    counts = [int(first[m + 1] - first[m]) for m in range(B)]
    for m in range(B):
        records[m].append({"stage": "build_graph", "vertices": int(valid_per_map[m]),
                           "edges": int(stats[4]) if B == 1 else None, "wall_ms": 0.0})
        records[m].append({"stage": "form_components", "component_count": counts[m],
                           "wall_ms": comp_ms})
        records[m].append({"stage": "edge_coefficients", "degenerate_edges": None,
                           "wall_ms": coef_ms})

    t0 = time.perf_counter()
    total = int(first[B])
    passes = 2 if settings.refill_reweighted else 1
    z = None
    for pas in range(passes):
        # pass 2 (solver.py:237-238): same components, weights re-evaluated
        # with the bilateral factors at the filled state (edge_weights at z)
        wts = None if pas == 0 else _edge_weights(g, co, z, EW_BILATERAL, weights)
        z, fill_iters, fill_status = _fill(g, labels, total, co, settings, wts)
        capped = np.flatnonzero(fill_status.cpu().numpy())
        for c in capped:
            m = int(np.searchsorted(first, c, side="right") - 1)
            warnings[m].append(f"component {int(c - first[m])}: cg hit iteration cap")
    if B == 1:
        records[0][2]["degenerate_edges"] = int(g.stats[5].item())
    else:
        _per_map_edge_stats(g, co[3], records)
    report = _lib.fill_report()
    if _FILL_SOLVER != "cg":
        report["mg"] = _lib.mg_report()
        report["mg_profile"] = _lib.mg_profile()
    fill_ms = _ms(t0)
    for m in range(B):
        records[m].append({"stage": "fill", "wall_ms": fill_ms})
    # the filled state (a copy: the outer loop updates z in place), 0 outside the mask
    filled = torch.where(g.nmap.valid_t.bool(), z, torch.zeros((), dtype=z.dtype, device=g.dev))
    fit = fill_iters.cpu().numpy()

    valid = g.nmap.valid_t
    loop = _BatchLoop(g, labels, first, counts, co, settings, weights)
    loop.defer_scales()
    loop.initial_keys()
    loop.build()
    active = np.arange(B, dtype=np.int32)
    e_prev = np.full(B, ENERGY_FLOOR)
    energies = [[] for _ in range(B)]
    iters = np.zeros(B, dtype=np.int64)
    version = np.zeros(B, dtype=np.int64)
    hasher = None
    chunk = _DeviceLoop(g, settings)
    deferred = []
    t = 0
    while len(active):
        # iterations that cannot merge run back to back with the convergence
        # test on the device (one read-back per chunk instead of per iteration)
        k = chunk.length(t)
        if k >= 2:
            chunk.sync_prev(e_prev)
            t = chunk.run(loop, z, t, k, active)
            still, finish = chunk.collect(loop, active, t, e_prev, energies, records, warnings,
                                          iters)
            active = np.array(still, dtype=np.int32)
            if len(active):
                finish()
            else:  # the loop is over: the records wait until the gauge is enqueued
                deferred.append(finish)
            continue
        it_start = time.perf_counter()
        residual, wts = loop.step(z, t, active)
        t_step = t
        t += 1
        merging = np.array([m for m in active
                            if settings.freq_merging is not None and t % settings.freq_merging == 0
                            and loop.count[m] > 1 and loop.map_edges[m] > 0], dtype=np.int32)
        digests = {}
        if len(merging):
            # merges relabel only, so z (and its digest) is the same before
            # and after; hash a device snapshot off the critical path
            loop.fold_scales(z, merging)  # the digests and the relabel see the applied z
            if hasher is None:
                hasher = cf.ThreadPoolExecutor(max_workers=4)
            snaps = {int(m): z[m * g.hw:(m + 1) * g.hw].clone() for m in merging}
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(g.dev))
            digests = {m: hasher.submit(_digest_async, snp, ready) for m, snp in snaps.items()}
            loop.merge(residual, wts, merging)
        # one read-back per iteration for every map
        host = torch.cat([loop.energy, loop.ok.to(torch.float64), loop.merge_energy,
                          loop.new_count.to(torch.float64)]).cpu().numpy()
        e_step, ok, e_merge, new_count = host[:B], host[B:2 * B], host[2 * B:3 * B], host[3 * B:]
        wall = _ms(it_start)
        merged = set(int(m) for m in merging)
        still = []
        for m in active:
            m = int(m)
            if not ok[m]:
                warnings[m].append(f"iteration {t_step}: cg hit iteration cap")
            extra = {}
            if m in merged:
                nc = int(new_count[m])
                e_t = float(e_merge[m])
                extra = {"components_before": int(loop.count[m]), "components_after": nc,
                         "z_digest_before": digests[m], "z_digest_after": digests[m]}
                loop.count[m] = nc
                version[m] += 1
            else:
                e_t = float(e_step[m])
            converged = _has_converged(e_t, e_prev[m], t, settings)
            e_prev[m] = e_t
            energies[m].append(e_t)
            records[m].append({"t": t, "E_t": e_t, "component_count": int(loop.count[m]),
                               "merge_performed": m in merged, "wall_ms": wall, **extra})
            if converged:
                iters[m] = t
            else:
                still.append(m)
        # a merge changes the quotient; maps that merely left the loop keep
        # their edges in it (every stage restricts itself to the active maps)
        if len(still) and merged:
            keep = np.zeros(B, dtype=bool)
            keep[still] = True
            loop.filter_keys(keep)
            loop.build()
        active = np.array(still, dtype=np.int32)

    loop.fold_scales(z, np.arange(B, dtype=np.int32))
    if hasher is not None:  # resolve the merge digests (pipeline.py:194-209)
        for recs in records:
            for r in recs:
                for key in ("z_digest_before", "z_digest_after"):
                    if key in r and isinstance(r[key], cf.Future):
                        r[key] = r[key].result()
        hasher.shutdown()
    target = 0.0 if gauge_depth is None else float(np.log(gauge_depth))
    lib = g.lib
    ws = _ws(_lib.size_query(lib.ni_gauge_workspace_size, g.B, g.H, g.W), g.dev)
    _lib.check(lib.ni_gauge(_ptr(z), _ptr(valid), g.B, g.H, g.W, C.c_double(target), C.c_void_p(0),
                            _ptr(ws), ws.numel(), g.s()), "gauge")
    for finish in deferred:
        finish()
    out = []
    for m in range(B):
        sl = slice(m * g.hw, (m + 1) * g.hw)
        records[m].append({"stage": "done", "iterations": int(iters[m]),
                           "warnings": len(warnings[m]), "wall_ms": _ms(run_start)})
        vm = valid[sl]
        out.append(PipelineResult(
            log_depth=LogDepthMap(z[sl], vm, g.H, g.W),
            filled=LogDepthMap(filled[sl], vm, g.H, g.W),
            partition0=Partition(labels0[sl], counts[m], 0, int(first[m])),
            partition=Partition(labels[sl], int(loop.count[m]), int(version[m]), int(first[m])),
            records=records[m],
            warnings=warnings[m],
            iterations=int(iters[m]),
            energies=energies[m],
            fill_iterations=fit[first[m]:first[m + 1]],
            fill_report=report,
        ))
    return out


_D2H_CTAS = 2  # read-back kernel CTAs (512 threads each); 0: copy engine.  Measured on the 64-map
# C5 stream (scripts/e2e_ab.py): 1-3 CTAs 65.5-67 ms per step, 16 CTAs 71-74 ms (a wide read-back
# kernel slows the concurrent compute kernels), copy engine 83 ms; 2 CTAs still finish the
# 537 MB well inside one step.
_D2H_PRIORITY = -1  # stream priority of the read-back kernel
_D2H_CTAS_LAST = 16  # the stream's last batch: nothing computes beside its read-back
_H2D_CTAS = 0  # upload kernel CTAs (ni_copy_from_host); 0: copy engine
_PIN_ALLOC_MS: list = []  # host time of the last pinned read-back allocations
_STREAMS: dict = {}  # (device, read-back priority) -> (upload stream, read-back stream)


def run_pipeline_stream(
    batches,
    intrinsics,
    theta_c: float | None,
    settings: SolveSettings | None = None,
    weights: WeightParams | None = None,
    connectivity: int = 8,
    model: str = "milano",
    gauge_depth: float | None = None,
    device=None,
):
    """Serve a stream of host batches through :func:`run_pipeline_batch`.

    ``batches`` yields ``(normals, mask)`` CPU tensors of shape (B, H, W, 3) /
    (B, H, W) (pinned memory lets the copies run asynchronously); every batch
    uses ``intrinsics`` (one per map).  Yields ``(results, log_depth_host)``
    per batch: the list of :class:`PipelineResult` and a pinned (B, H*W)
    float64 CPU tensor with every map's log-depth (0 outside the mask).

    The next batch's host->device copy and the previous batch's log-depth
    read-back run on two copy streams while the current batch computes, so a
    stream of batches pays for the transfers only at its two ends.  The
    results are those of ``run_pipeline_batch`` on each batch.
    """
    dev = _device(device)
    comp = torch.cuda.current_stream(dev)
    # The two copy streams are made once per device: torch's caching allocator
    # pools blocks per stream, so fresh streams per call would re-allocate the
    # 0.9 GB upload buffers with cudaMalloc every time (measured: the first
    # batch of some streams took 60-300 ms longer) and strand the old ones.
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), _D2H_PRIORITY)
    if key not in _STREAMS:
        _STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev, priority=_D2H_PRIORITY))
    h2d, d2h = _STREAMS[key]
    # uploads and read-backs on separate streams: the
    # link is full duplex, so they overlap each other too.  The read-back is a
    # small SM kernel storing into mapped pinned memory (ni_copy_to_host), not a
    # copy-engine transfer: a ~10 ms copy-engine read-back would hold the
    # device->host queue that every small control read (.cpu()) of the next
    # batch's pipeline waits in.  High priority: its few CTAs are scheduled
    # ahead of the compute grids' pending CTAs.
    lib = _lib.load()
    it = iter(batches)

    # Two pairs of upload buffers, used in turn: NormalMap.create has consumed a
    # pair (and synchronised) before the batch computes, so the next-but-one
    # upload can overwrite it.  Allocating the buffers per batch instead left
    # their reuse to the caching allocator's cross-stream bookkeeping, which
    # sometimes had to cudaMalloc 0.9 GB in the middle of the stream (one bench
    # run in five lost 80-200 ms there).
    ring = [None, None]
    count = [0]

    def upload():
        try:
            n_h, m_h = next(it)
        except StopIteration:
            return None
        i = count[0] % 2
        count[0] += 1
        slot = ring[i]
        with torch.cuda.stream(h2d):
            if (slot is None or slot[0].shape != n_h.shape or slot[0].dtype != n_h.dtype
                    or slot[1].shape != m_h.shape or slot[1].dtype != m_h.dtype):
                slot = [torch.empty(n_h.shape, dtype=n_h.dtype, device=dev),
                        torch.empty(m_h.shape, dtype=m_h.dtype, device=dev), None]
                ring[i] = slot
            elif slot[2] is not None:
                h2d.wait_event(slot[2])  # the batch that used this pair has been ingested
            n_d, m_d = slot[0], slot[1]
            if (_H2D_CTAS and not n_h.is_cuda
                    and all(t.is_pinned() and t.is_contiguous() for t in (n_h, m_h))):
                # upload by a small SM kernel reading the mapped pinned buffers
                # (ni_copy_from_host), like the read-back
                for d_t, h_t in ((n_d, n_h), (m_d, m_h)):
                    _lib.check(lib.ni_copy_from_host(
                        C.c_void_p(d_t.data_ptr()), C.c_void_p(h_t.data_ptr()),
                        h_t.numel() * h_t.element_size(), _H2D_CTAS,
                        C.c_void_p(h2d.cuda_stream)), "upload")
            else:
                n_d.copy_(n_h, non_blocking=True)
                m_d.copy_(m_h, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(h2d)
        return n_d, m_d, ready, slot

    nxt = upload()
    try:
        yield from _stream_loop(nxt, upload, comp, d2h, lib, dev, intrinsics, theta_c, settings,
                                weights, connectivity, model, gauge_depth)
    finally:  # a consumer that stops early: the read-back kernel may still write `out`
        d2h.synchronize()


def _stream_loop(nxt, upload, comp, d2h, lib, dev, intrinsics, theta_c, settings, weights,
                 connectivity, model, gauge_depth):
    pending = None
    while nxt is not None:
        n_d, m_d, ready, slot = nxt
        comp.wait_event(ready)
        nxt = upload()  # prefetch the next batch while this one computes
        nmap = NormalMap.create(n_d, m_d, device=dev)
        slot[2] = torch.cuda.Event()  # the upload pair is free again
        slot[2].record(comp)
        res = run_pipeline_batch(nmap, intrinsics, theta_c, settings, weights, connectivity,
                                 model, gauge_depth)
        del nmap
        done = torch.cuda.Event()
        done.record(comp)
        t_alloc = time.perf_counter()
        out = torch.empty((len(res), res[0].log_depth.height * res[0].log_depth.width),
                          dtype=torch.float64, pin_memory=True)
        _PIN_ALLOC_MS.append(_ms(t_alloc))  # diagnostic (scripts/e2e_outlier.py)
        del _PIN_ALLOC_MS[:-64]
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            hw = out.shape[1]
            vals = [r.log_depth.values_t for r in res]
            base = vals[0].data_ptr()
            whole = all(v.is_contiguous() and v.data_ptr() == base + 8 * hw * i
                        for i, v in enumerate(vals))  # the batch's z: one copy
            for i, v in enumerate(vals):
                v.record_stream(d2h)
                if not _D2H_CTAS:  # copy-engine read-back (the A/B baseline)
                    out[i].copy_(v, non_blocking=True)
                    continue
                if whole and i:
                    continue
                nbytes = 8 * hw * (len(vals) if whole else 1)
                ctas = _D2H_CTAS if nxt is not None else max(_D2H_CTAS, _D2H_CTAS_LAST)
                _lib.check(lib.ni_copy_to_host(C.c_void_p(v.data_ptr()),
                                               C.c_void_p(out[i].data_ptr()), nbytes,
                                               ctas, C.c_void_p(d2h.cuda_stream)),
                           "read-back")
            fetched = torch.cuda.Event()
            fetched.record(d2h)
        if pending is not None:
            pending[2].synchronize()
            yield pending[0], pending[1]
        pending = (res, out, fetched)
    if pending is not None:
        pending[2].synchronize()
        yield pending[0], pending[1]


def _per_map_edge_stats(g: _Grid, eflags: torch.Tensor, records):
    """Per-map edge / degenerate counts for batched runs (records of
    pipeline.py:137-159 are per map), counted by the coefficients kernel."""
    cnt = g.map_counts.view(g.B, 2).cpu().numpy()
    ex, dg = cnt[:, 0], cnt[:, 1]
    for m in range(g.B):
        records[m][0]["edges"] = int(ex[m])
        records[m][2]["degenerate_edges"] = int(dg[m])


def run_pipeline(
    nmap: NormalMap,
    intr: CameraIntrinsics,
    theta_c: float | None,
    settings: SolveSettings | None = None,
    weights: WeightParams | None = None,
    connectivity: int = 8,
    model: str = "milano",
    gauge_depth: float | None = None,
) -> PipelineResult:
    """Reconstruct a log-depth map from a normal map via component scales.

    Same contract as normint.run_pipeline (pipeline.py:105-248): ``theta_c``
    in radians (None = per-pixel components), output gauge-fixed to unit
    median depth unless ``gauge_depth`` is given.  Numerical differences
    (INTEGRATION.md): the fill is solved by a multigrid-preconditioned fp32
    CG to scipy's tolerance, and the scale step removes the roundoff
    null-space part of its right-hand side -- a no-op unless the reference's
    own scale CG hits its cap, where the reference's records, warnings and
    energies follow a roundoff-driven trajectory these do not reproduce.
    """
    nmap = as_normal_map(nmap)
    if nmap.batch != 1:
        raise ValueError("run_pipeline takes a single map; use run_pipeline_batch")
    return run_pipeline_batch(nmap, [intr], theta_c, settings, weights, connectivity, model,
                              gauge_depth)[0]


@dataclass
class BaselineResult:
    """pipeline.py:288-294."""

    log_depth: LogDepthMap
    records: list
    warnings: list = field(default_factory=list)
    iterations: int = 0
    energies: list = field(default_factory=list)


def run_pixel_baseline_batch(
    nmap: NormalMap,
    intrinsics,
    settings: SolveSettings | None = None,
    weights: WeightParams | None = None,
    connectivity: int = 8,
    model: str = "milano",
    gauge_depth: float | None = None,
) -> list[BaselineResult]:
    """``run_pixel_baseline`` (pipeline.py:297-369) over the B maps of a batch.

    Each outer iteration re-solves the full pixel system of every map that has
    not converged -- one CG per map over all its valid pixels, from x0 = 0,
    with the inter-system weight schedule (pipeline.py:261-285) -- in one
    batched weighted-fill launch, and the solutions replace z.
    """
    settings = as_settings(settings) or SolveSettings()
    weights = as_weights(weights) or WeightParams()
    _validate(model, connectivity)
    nmap = as_normal_map(nmap)
    B = nmap.batch
    intr = list(intrinsics) if isinstance(intrinsics, (list, tuple)) else [intrinsics] * B
    intr = [as_intrinsics(i) for i in intr]
    if len(intr) != B:
        raise ValueError("need one CameraIntrinsics per map")
    run_start = time.perf_counter()
    g = _Grid(nmap, connectivity, model)
    if nmap.valid_count == 0:
        raise EmptyMask("normal map has no valid pixel")
    co = _coefficients(g, intr)
    valid = g.nmap.valid_t
    vbool = valid.bool()
    nvalid = valid.view(B, -1).sum(dim=1, dtype=torch.int64).cpu().numpy()
    if (nvalid == 0).any():  # every map raises like the reference (graph.py:65-66)
        raise EmptyMask("normal map has no valid pixel")
    mapid = (torch.arange(g.npix, device=g.dev, dtype=torch.int64) // g.hw).to(torch.int32)
    z = torch.zeros(g.npix, dtype=torch.float64, device=g.dev)
    records = [[] for _ in range(B)]
    warnings = [[] for _ in range(B)]
    energies = [[] for _ in range(B)]
    iters = np.zeros(B, dtype=np.int64)
    e_prev = np.full(B, ENERGY_FLOOR)
    active = np.ones(B, dtype=bool)
    t = 0
    while active.any():
        it_start = time.perf_counter()
        act_t = torch.from_numpy(active).to(g.dev)
        live = vbool & act_t[mapid.long()]
        labels = torch.where(live, mapid, torch.full_like(mapid, -1))
        wts = _edge_weights(g, co, z, EW_UNIFORM if t < settings.alignment_iters else EW_FULL,
                            weights)
        x, _, status = _fill(g, labels, B, co, settings, wts)
        energy = _pair_energy(g, co, x, wts)
        z = torch.where(live, x, z)
        host = torch.cat([energy, status.to(torch.float64)]).cpu().numpy()
        e_now, capped = host[:B], host[B:]
        wall = _ms(it_start)
        t_step = t
        t += 1
        for m in np.flatnonzero(active):
            m = int(m)
            if capped[m]:
                warnings[m].append(f"iteration {t_step}: cg hit iteration cap")
            e_t = float(e_now[m])
            conv = _has_converged(e_t, e_prev[m], t, settings)
            e_prev[m] = e_t
            energies[m].append(e_t)
            records[m].append({"t": t, "E_t": e_t, "component_count": int(nvalid[m]),
                               "merge_performed": False, "wall_ms": wall})
            if conv:
                active[m] = False
                iters[m] = t
    target = 0.0 if gauge_depth is None else float(np.log(gauge_depth))
    ws = _ws(_lib.size_query(g.lib.ni_gauge_workspace_size, g.B, g.H, g.W), g.dev)
    _lib.check(g.lib.ni_gauge(_ptr(z), _ptr(valid), g.B, g.H, g.W, C.c_double(target),
                              C.c_void_p(0), _ptr(ws), ws.numel(), g.s()), "gauge")
    out = []
    for m in range(B):
        sl = slice(m * g.hw, (m + 1) * g.hw)
        records[m].append({"stage": "done", "iterations": int(iters[m]),
                           "warnings": len(warnings[m]), "wall_ms": _ms(run_start)})
        out.append(BaselineResult(LogDepthMap(z[sl], valid[sl], g.H, g.W), records[m],
                                  warnings[m], int(iters[m]), energies[m]))
    return out


def run_pixel_baseline(
    nmap: NormalMap,
    intr: CameraIntrinsics,
    settings: SolveSettings | None = None,
    weights: WeightParams | None = None,
    connectivity: int = 8,
    model: str = "milano",
    gauge_depth: float | None = None,
) -> BaselineResult:
    """Iteratively reweighted per-pixel log-depth integration
    (pipeline.py:297-369): same weight schedule and convergence test as
    ``run_pipeline``, but the full pixel system is re-solved every iteration."""
    nmap = as_normal_map(nmap)
    if nmap.batch != 1:
        raise ValueError("run_pixel_baseline takes a single map; use run_pixel_baseline_batch")
    return run_pixel_baseline_batch(nmap, [intr], settings, weights, connectivity, model,
                                    gauge_depth)[0]


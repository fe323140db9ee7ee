"""The reference's internal seams, with its signatures, on the B200 kernels.

``normint`` exposes the stages of ``run_pipeline`` as separate functions
(SURVEY.md 8(b)); code written against them keeps working here:

* ``build_pixel_graph(nmap, connectivity)``            graph.py:56-86
* ``form_components(g, nmap, theta_c)``                graph.py:141-165
* ``build_edge_coefficients(nmap, g, intr, model)``    continuity.py:210-289
* ``fill_components(p, g, coeffs, params, settings)``  solver.py:195-239
* ``build_quotient(g, p)``                             graph.py:186-196
* ``relative_scale_step(q, p, z, t, settings, params, coeffs)``  solver.py:281-303
* ``merge_components(q, p, residuals)``                graph.py:207-250
* ``apply_scales(zmap, p, scales)``                    solver.py:306-313

Each one runs the same C-ABI entry point ``run_pipeline`` uses, on one map.
Graph-level data stays in the grid layout on the device (edges are implicit:
forward edge k of pixel i, key ``i * KF + k``, and ascending keys are exactly
the reference's lexicographic edge order); the reference's per-edge numpy
arrays (``edges``, ``omega_to_a`` ...) are materialised lazily on first
access.  Reference objects (``normint.NormalMap``, ``Partition``,
``EdgeCoefficients`` ...) are accepted wherever the reference takes them.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import EmptyMask
from .geometry import LogDepthMap, NormalMap, as_intrinsics, as_normal_map
from .pipeline import (EW_BILATERAL, Partition, _BatchLoop, _coefficients, _components,
                       _edge_weights, _fill, _Grid, _ptr, _validate, _ws)
from .settings import SolveSettings, WeightParams, as_settings, as_weights

# forward offsets (du, dv) in key order k (graph.py:24-25)
OFFSETS = {4: ((1, 0), (0, 1)), 8: ((1, 0), (-1, 1), (0, 1), (1, 1))}


def _lazy_np(t: torch.Tensor) -> np.ndarray:
    a = t.cpu().numpy()
    a.flags.writeable = False
    return a


# ------------------------------------------------------------------- graph


class PixelGraph:
    """Adjacency of the valid pixels (graph.py:29-53), implicit in the grid.

    ``eflags_t`` (device, uint8 per pixel): bit k set iff forward edge k joins
    two valid pixels.  ``keys_t`` (device, int64): ``pixel * KF + k`` of every
    edge, ascending = the reference's edge order.
    """

    def __init__(self, nmap: NormalMap, connectivity: int):
        self.nmap = nmap
        self.width, self.height = nmap.width, nmap.height
        self.connectivity = int(connectivity)
        self.kf = len(OFFSETS[self.connectivity])
        h, w = self.height, self.width
        v = nmap.valid_t.view(h, w).bool()
        bits = torch.zeros((h, w), dtype=torch.uint8, device=nmap.device)
        for k, (du, dv) in enumerate(OFFSETS[self.connectivity]):
            pair = torch.zeros_like(v)
            src_u = slice(max(0, -du), w - max(0, du))
            dst_u = slice(max(0, du), w + min(0, du))
            pair[0:h - dv, src_u] = v[0:h - dv, src_u] & v[dv:h, dst_u]
            bits |= pair.to(torch.uint8) << k
        self.eflags_t = bits.view(-1).contiguous()
        self._keys = None
        self._edges = None
        self._vertices = None

    @property
    def keys_t(self) -> torch.Tensor:
        if self._keys is None:
            sh = torch.arange(self.kf, device=self.eflags_t.device, dtype=torch.uint8)
            has = ((self.eflags_t[:, None] >> sh[None, :]) & 1).bool().view(-1)
            self._keys = torch.nonzero(has).view(-1)
        return self._keys

    def _endpoints(self, keys: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        off = torch.tensor([dv * self.width + du for du, dv in OFFSETS[self.connectivity]],
                           dtype=torch.int64, device=keys.device)
        a = keys // self.kf
        return a, a + off[keys % self.kf]

    @property
    def edges(self) -> np.ndarray:
        """(E, 2) int64 pixel ids, a < b, lexicographically sorted."""
        if self._edges is None:
            a, b = self._endpoints(self.keys_t)
            self._edges = _lazy_np(torch.stack([a, b], dim=1))
        return self._edges

    @property
    def vertices(self) -> np.ndarray:
        if self._vertices is None:
            self._vertices = _lazy_np(torch.nonzero(self.nmap.valid_t).view(-1))
        return self._vertices

    @property
    def vertex_count(self) -> int:
        return self.nmap.valid_count

    @property
    def edge_count(self) -> int:
        return int(self.keys_t.numel())

    @property
    def compact_index(self) -> np.ndarray:
        idx = np.full(self.width * self.height, -1, dtype=np.int64)
        idx[self.vertices] = np.arange(len(self.vertices))
        return idx


def build_pixel_graph(nmap, connectivity: int = 8) -> PixelGraph:
    """graph.py:56-86: raises EmptyMask without a valid pixel."""
    if connectivity not in (4, 8):
        raise ValueError("connectivity must be 4 or 8")
    nmap = as_normal_map(nmap)
    if nmap.batch != 1:
        raise ValueError("build_pixel_graph takes a single map")
    if nmap.valid_count == 0:
        raise EmptyMask("normal map has no valid pixel")
    return PixelGraph(nmap, connectivity)


def _as_graph(g, nmap=None) -> PixelGraph:
    if isinstance(g, PixelGraph):
        return g
    # a reference PixelGraph: rebuild the implicit one from the map it came from
    if nmap is None:
        raise TypeError("a reference PixelGraph needs its NormalMap")
    return build_pixel_graph(nmap, g.connectivity)


def _as_partition(p, dev) -> Partition:
    if isinstance(p, Partition):
        return p
    lab = torch.from_numpy(np.asarray(p.labels).astype(np.int32)).to(dev)
    return Partition(lab, int(p.component_count), int(getattr(p, "version", 0)))


def form_components(g, nmap, theta_c: float | None) -> Partition:
    """graph.py:141-165: connected components of the edges with relative
    normal angle < theta_c (radians; None = one component per pixel),
    canonically labelled (ni_components)."""
    nmap = as_normal_map(nmap)
    g = _as_graph(g, nmap)
    grid = _Grid(nmap, g.connectivity, "milano")
    labels, map_first = _components(grid, theta_c)
    return Partition(labels, int(map_first[1].item()))


# ------------------------------------------------------------ coefficients


class EdgeCoefficients:
    """Per-edge coefficients (continuity.py:166-189) over the grid planes.

    ``planes`` = (omega_a (KF, N), omega_b (KF, N) or None, gamma (N,),
    eflags (N,)) as ``ni_coefficients`` writes them; the reference's per-edge
    arrays (indexed like ``graph.edges``) are materialised on first access.
    """

    def __init__(self, g: PixelGraph, planes, model: str):
        self.graph = g
        self.planes = planes
        self.model = model
        self._host = {}

    @property
    def edge_count(self) -> int:
        return self.graph.edge_count

    def _arrays(self) -> dict:
        if not self._host:
            g = self.graph
            omega_a, omega_b, gamma, eflags = self.planes
            keys = g.keys_t
            a, b = g._endpoints(keys)
            k = keys % g.kf
            oa = omega_a[k, a]
            ob = omega_b[k, a] if omega_b is not None else -oa
            valid = ((eflags[a] >> (4 + k).to(torch.uint8)) & 1).bool()
            h, w = g.height, g.width
            du = torch.tensor([o[0] for o in OFFSETS[g.connectivity]], device=keys.device)[k]
            dv = torch.tensor([o[1] for o in OFFSETS[g.connectivity]], device=keys.device)[k]
            vmask = g.nmap.valid_t.bool()

            def reflect(center, sgn):  # continuity.py:196-207
                cu, cv = center % w, center // w
                ru, rv = cu + sgn * du, cv + sgn * dv
                inside = (ru >= 0) & (ru < w) & (rv >= 0) & (rv < h)
                ids = torch.where(inside, rv * w + ru, torch.zeros_like(ru))
                return torch.where(inside & vmask[ids], ids, torch.full_like(ids, -1))

            self._host = {
                "edges": g.edges,
                "omega_to_a": _lazy_np(oa), "omega_to_b": _lazy_np(ob),
                "gamma_a": _lazy_np(gamma[a]), "gamma_b": _lazy_np(gamma[b]),
                "opp_a": _lazy_np(reflect(a, -1)), "opp_b": _lazy_np(reflect(b, 1)),
                "valid": _lazy_np(valid),
            }
        return self._host

    def __getattr__(self, name):
        if name in ("edges", "omega_to_a", "omega_to_b", "gamma_a", "gamma_b", "opp_a", "opp_b",
                    "valid"):
            return self._arrays()[name]
        raise AttributeError(name)


def build_edge_coefficients(nmap, g, intr, model: str = "milano") -> EdgeCoefficients:
    """continuity.py:210-289 (ni_coefficients): Milano (4/8-conn) or BiNI
    (4-conn) log-depth differences, per-pixel gamma, validity."""
    nmap = as_normal_map(nmap)
    g = _as_graph(g, nmap)
    _validate(model, g.connectivity)
    grid = _Grid(nmap, g.connectivity, model)
    return EdgeCoefficients(g, _coefficients(grid, [as_intrinsics(intr)]), model)


def _planes(coeffs, g: PixelGraph):
    """Grid planes of our EdgeCoefficients, or scattered from a reference one."""
    if isinstance(coeffs, EdgeCoefficients):
        return coeffs.planes
    dev = g.nmap.device
    n = g.width * g.height
    keys = g.keys_t
    a, b = g._endpoints(keys)
    k = keys % g.kf
    f64 = lambda x: torch.from_numpy(np.asarray(x, dtype=np.float64)).to(dev)  # noqa: E731
    omega_a = torch.zeros((g.kf, n), dtype=torch.float64, device=dev)
    omega_a[k, a] = f64(coeffs.omega_to_a)
    omega_b = None
    if coeffs.model == "bini":
        omega_b = torch.zeros((g.kf, n), dtype=torch.float64, device=dev)
        omega_b[k, a] = f64(coeffs.omega_to_b)
    gamma = torch.zeros(n, dtype=torch.float64, device=dev)
    gamma[a] = f64(coeffs.gamma_a)
    gamma[b] = f64(coeffs.gamma_b)
    vbit = torch.from_numpy(np.asarray(coeffs.valid, dtype=bool)).to(dev).to(torch.int32)
    ef = g.eflags_t.to(torch.int32).clone()
    ef.index_add_(0, a, vbit << (4 + k).to(torch.int32))
    return omega_a, omega_b, gamma, ef.to(torch.uint8)


def _grid_for(g: PixelGraph, coeffs) -> _Grid:
    return _Grid(g.nmap, g.connectivity, getattr(coeffs, "model", "milano"))


# -------------------------------------------------------------------- fill


def fill_components(p, g, coeffs, params=None, settings=None) -> tuple[np.ndarray, list[str]]:
    """solver.py:195-239: every component reconstructed from zero log-depth
    (one batched multigrid-preconditioned CG, ni_fill_mg), plus the optional
    reweighted second pass.  Returns the flattened full-grid log-depth (0
    outside the mask and for single-pixel components) and cap warnings."""
    params = as_weights(params) or WeightParams()
    settings = as_settings(settings) or SolveSettings()
    g = _as_graph(g, getattr(coeffs, "graph", None) and coeffs.graph.nmap)
    grid = _grid_for(g, coeffs)
    co = _planes(coeffs, g)
    p = _as_partition(p, grid.dev)
    warnings: list[str] = []
    z = None
    for pas in range(2 if settings.refill_reweighted else 1):
        wts = None if pas == 0 else _edge_weights(grid, co, z, EW_BILATERAL, params)
        z, _, status = _fill(grid, p.labels_t, p.component_count, co, settings, wts)
        for c in np.flatnonzero(status.cpu().numpy()):
            warnings.append(f"component {int(c)}: cg hit iteration cap")
    z = torch.where(g.nmap.valid_t.bool(), z, torch.zeros((), dtype=z.dtype, device=grid.dev))
    return z.cpu().numpy(), warnings


# ---------------------------------------------------------------- quotient


class QuotientGraph:
    """Component-level view (graph.py:168-183): the inter-component edges of
    the pixel graph, in edge order.  ``keys_t`` (device int32) are their grid
    keys; the reference arrays are materialised on first access."""

    def __init__(self, g: PixelGraph, p: Partition, keys_t: torch.Tensor):
        self.graph = g
        self.partition = p
        self.component_count = p.component_count
        self.keys_t = keys_t
        self._host = {}

    @property
    def inter_edge_count(self) -> int:
        return int(self.keys_t.numel())

    def _arrays(self) -> dict:
        if not self._host:
            g = self.graph
            keys = self.keys_t.to(torch.int64)
            a, b = g._endpoints(keys)
            lab = self.partition.labels_t.to(torch.int64)
            self._host = {
                "inter_edges": _lazy_np(torch.stack([a, b], dim=1)),
                "edge_ids": _lazy_np(torch.searchsorted(g.keys_t, keys)),
                "comp_pairs": _lazy_np(torch.stack([lab[a], lab[b]], dim=1)),
            }
        return self._host

    def __getattr__(self, name):
        if name in ("inter_edges", "edge_ids", "comp_pairs"):
            return self._arrays()[name]
        raise AttributeError(name)


def build_quotient(g, p) -> QuotientGraph:
    """graph.py:186-196 (ni_inter_edges): edges whose endpoints lie in
    different components, in edge order."""
    g = _as_graph(g)
    grid = _Grid(g.nmap, g.connectivity, "milano")
    p = _as_partition(p, grid.dev)
    lib = grid.lib
    out = torch.empty(max(grid.npix * grid.kf, 1), dtype=torch.int32, device=grid.dev)
    n = torch.zeros(1, dtype=torch.int32, device=grid.dev)
    ws = _ws(_lib.size_query(lib.ni_inter_edges_workspace_size, 1, grid.H, grid.W, grid.conn),
             grid.dev)
    eflags = g.eflags_t  # existence bits only: all ni_inter_edges reads
    _lib.check(lib.ni_inter_edges(_ptr(p.labels_t), _ptr(eflags), 1, grid.H, grid.W, grid.conn,
                                  _ptr(out), _ptr(n), _ptr(ws), ws.numel(), grid.s()),
               "build_quotient")
    return QuotientGraph(g, p, out[:int(n.item())].clone())


def _loop_for(q: QuotientGraph, p: Partition, coeffs, settings, params, labels=None):
    g = q.graph
    grid = _grid_for(g, coeffs)
    co = None if coeffs is None else _planes(coeffs, g)  # the merge reads no coefficients
    lab = p.labels_t if labels is None else labels
    loop = _BatchLoop(grid, lab, np.array([0, p.component_count]), [p.component_count], co,
                      settings, params)
    loop.keys = q.keys_t
    loop.K = q.inter_edge_count
    loop.build()
    return loop


class ScaleStep:
    """Outcome of one relative-scale iteration (solver.py:242-250)."""

    def __init__(self, scales, energy, residual, weights, cg_converged):
        self.scales = scales
        self.energy = float(energy)
        self.residual = residual
        self.weights = weights
        self.cg_converged = bool(cg_converged)


def relative_scale_step(q, p, z_flat, t: int, settings=None, params=None,
                        coeffs=None) -> ScaleStep:
    """solver.py:281-303 (ni_scale_step): inter-edge weights for iteration t,
    the relative-scale CG, row residuals A s - b and the weighted energy.
    ``z_flat`` is not modified (the kernel's in-place apply runs on a copy)."""
    settings = as_settings(settings) or SolveSettings()
    params = as_weights(params) or WeightParams()
    if not isinstance(q, QuotientGraph):
        raise TypeError("relative_scale_step needs a QuotientGraph from build_quotient")
    p = _as_partition(p, q.graph.nmap.device)
    if q.inter_edge_count == 0:
        return ScaleStep(np.zeros(p.component_count), 0.0, np.zeros(0), np.zeros(0), True)
    loop = _loop_for(q, p, coeffs, settings, params)
    z = torch.as_tensor(np.asarray(z_flat, dtype=np.float64)).to(loop.g.dev).clone()
    residual, wts = loop.step(z, int(t), np.array([0], dtype=np.int32))
    k2 = 2 * q.inter_edge_count
    host = torch.cat([loop.energy[:1], loop.ok[:1].to(torch.float64)]).cpu().numpy()
    return ScaleStep(loop.last_scales[:p.component_count].cpu().numpy(), host[0],
                     residual[:k2].cpu().numpy(), wts[:k2].cpu().numpy(), host[1] != 0)


def merge_components(q, p, residuals) -> Partition:
    """graph.py:207-250 (ni_merge): every component joins its smallest-
    residual neighbour (ties by edge order); new canonical labels."""
    residuals = np.asarray(residuals, dtype=np.float64)
    if not isinstance(q, QuotientGraph):
        raise TypeError("merge_components needs a QuotientGraph from build_quotient")
    if residuals.shape != (q.inter_edge_count,):
        raise ValueError("need one residual per inter-edge")
    if not np.all(np.isfinite(residuals)):
        raise ValueError("residuals must be finite")
    p = _as_partition(p, q.graph.nmap.device)
    if q.inter_edge_count == 0:
        return Partition(p.labels_t, p.component_count, p.version + 1)
    labels = p.labels_t.clone()  # ni_merge relabels in place
    loop = _loop_for(q, p, None, SolveSettings(), WeightParams(), labels)
    dev = loop.g.dev
    res2 = torch.zeros(2 * q.inter_edge_count, dtype=torch.float64, device=dev)
    res2[0::2] = torch.from_numpy(residuals).to(dev)  # the merge key is |residual[2e]|
    loop.merge(res2, torch.zeros_like(res2), np.array([0], dtype=np.int32))
    return Partition(labels, int(loop.new_count[0].item()), p.version + 1)


def apply_scales(zmap: LogDepthMap, p, scales) -> LogDepthMap:
    """solver.py:306-313: every valid pixel shifted by its component's scale."""
    p = _as_partition(p, zmap.values_t.device)
    s = torch.as_tensor(np.asarray(scales, dtype=np.float64)).to(zmap.values_t.device)
    if s.numel() != p.component_count:
        raise ValueError("one scale per component required")
    lab = p.labels_t.to(torch.int64)
    ok = lab >= 0
    v = zmap.values_t + torch.where(ok, s[lab.clamp(min=0)], torch.zeros_like(zmap.values_t))
    return LogDepthMap(v, zmap.mask_t, zmap.height, zmap.width)


__all__ = ["PixelGraph", "EdgeCoefficients", "QuotientGraph", "ScaleStep", "build_pixel_graph",
           "form_components", "build_edge_coefficients", "fill_components", "build_quotient",
           "relative_scale_step", "merge_components", "apply_scales"]

"""CPU oracle for the component-based normal-integration hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this module, and only as the checker or as the timed CPU baseline.  The
product path (``paper_2510_11508_b200``) never imports it and has no CPU
fallback.

This is a numpy restatement of ``normint.run_pipeline`` (reference package
``/root/reference/pkg/src/normint``, v0.1.0).  Every function cites the
reference lines it follows.  The reference's arithmetic lives partly in
third-party code; those pieces are restated here from their published
algorithms and named with the versions installed in this image:

* ``scipy.sparse.linalg.cg`` (scipy 1.18.1, ``_isolve/iterative.py``):
  unpreconditioned CG, x0 = 0, stop when ||r|| < rtol * ||b|| checked at the
  top of each iteration, ``info = maxiter`` when the loop is exhausted.
  Restated in :func:`conjugate_gradient`.
* ``scipy.sparse.csgraph.connected_components`` (Cython): undirected
  connected components.  Restated as a vectorised union-find in
  :func:`_union_find_roots` (roots are the smallest member id, which is also
  the canonical label order of graph.py:133-138).
* ``scipy.special.expit``: logistic function, restated in :func:`_sigmoid`.
* scipy sparse CSR products (``A.T @ W @ A``): the normal matrix is assembled
  as the weighted graph Laplacian it equals and kept
  in a ``scipy.sparse.csr_matrix`` container for the matvec.

Parity of this restatement is pinned against the real reference by the
golden fixtures under ``tests/golden/`` (generated in the build container by
``tests/golden/make_golden.py``, which imports the reference), checked in
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import hashlib
import math
import struct
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

UNIT_NORM_TOL = 1e-4  # geometry.py:22
EPS_DEN = 1e-8  # continuity.py:34
EPS_LOG = 1e-12  # continuity.py:35
LOG_FLOOR = 1e-300  # continuity.py:36
ENERGY_FLOOR = 1e-300  # pipeline.py:55

OFFSETS = {4: ((1, 0), (0, 1)), 8: ((1, 0), (-1, 1), (0, 1), (1, 1))}  # graph.py:24-25


class OracleError(Exception):
    pass


class EmptyMaskError(OracleError):
    """Mirrors normint.errors.EmptyMask (graph.py:65-66)."""


@dataclass
class Settings:
    """Mirrors SolveSettings (solver.py:26-49) + WeightParams (continuity.py:42-57)."""

    cg_tol: float = 1e-6
    cg_max_iters: int = 5000
    delta_e_max: float = 1e-3
    max_iters: int = 150
    alignment_iters: int = 2
    freq_merging: int | None = None
    refill_reweighted: bool = False
    k: float = 2.0
    outlier_low: float = 1e-5
    outlier_high: float = 1e-3
    reweighting_mode: str = "soft"


# ---------------------------------------------------------------- geometry


def normalize_normals(normals, mask=None):
    """Validate and renormalise (geometry.py:115-145).

    float64 norm sqrt((x0^2 + x1^2) + x2^2), reject |norm - 1| > 1e-4 on valid
    pixels, divide, zero the invalid pixels.
    """
    n = np.asarray(normals, dtype=np.float64)
    if n.ndim != 3 or n.shape[2] != 3:
        raise ValueError("normals must have shape (H, W, 3)")
    m = np.ones(n.shape[:2], bool) if mask is None else np.asarray(mask, dtype=bool)
    if m.shape != n.shape[:2]:
        raise ValueError("mask shape does not match normals")
    if not np.all(np.isfinite(n[m])):
        raise ValueError("valid normals must be finite")
    sq = n * n
    norm = np.sqrt((sq[..., 0] + sq[..., 1]) + sq[..., 2])
    bad = m & (np.abs(norm - 1.0) > UNIT_NORM_TOL)
    if bad.any():
        raise ValueError(f"{int(bad.sum())} valid normals deviate from unit norm")
    out = np.zeros_like(n)
    out[m] = n[m] / norm[m][:, None]
    return out, m


def rays(fx, fy, cx, cy, u, v):
    """tau = ((u-cx)/fx, (v-cy)/fy, 1) (geometry.py:51-60)."""
    u = np.asarray(u, np.float64)
    v = np.asarray(v, np.float64)
    return np.stack([(u - cx) / fx, (v - cy) / fy, np.ones_like(u)], axis=-1)


# ------------------------------------------------------------------- graph


def pixel_edges(mask, connectivity=8):
    """Valid forward pairs, lexicographically ordered (graph.py:56-86).

    Returns ``(edges (E, 2) int64, direction (E,) int8)``; ``direction`` is
    the index into OFFSETS[connectivity].  For W > 2 the forward offsets are
    increasing in row-major id, so sorting by (a, direction) equals the
    reference's lexsort by (a, b).
    """
    if connectivity not in (4, 8):
        raise ValueError("connectivity must be 4 or 8")
    h, w = mask.shape
    if not mask.any():
        raise EmptyMaskError("normal map has no valid pixel")
    ids = np.arange(h * w, dtype=np.int64).reshape(h, w)
    a_l, b_l, d_l = [], [], []
    for k, (du, dv) in enumerate(OFFSETS[connectivity]):
        u0, u1 = max(0, -du), w - max(0, du)
        src = mask[0:h - dv, u0:u1]
        dst = mask[dv:h, u0 + du:u1 + du]
        both = src & dst
        a_l.append(ids[0:h - dv, u0:u1][both])
        b_l.append(ids[dv:h, u0 + du:u1 + du][both])
        d_l.append(np.full(int(both.sum()), k, np.int8))
    a = np.concatenate(a_l)
    b = np.concatenate(b_l)
    d = np.concatenate(d_l)
    order = np.lexsort((b, a))
    return np.stack([a[order], b[order]], axis=1), d[order]


def _union_find_roots(n, ea, eb):
    """Roots (= smallest member id) of the undirected graph (n nodes, edges
    ea-eb).  Hook the larger root under the smaller one, then compress; the
    minimum id of a set is always its root because parent[x] <= x."""
    parent = np.arange(n, dtype=np.int64)
    if len(ea) == 0:
        return parent
    ea = np.asarray(ea, np.int64)
    eb = np.asarray(eb, np.int64)
    while True:
        ra = parent[ea]
        rb = parent[eb]
        lo = np.minimum(ra, rb)
        hi = np.maximum(ra, rb)
        live = lo != hi
        if not live.any():
            return parent
        np.minimum.at(parent, hi[live], lo[live])
        while True:
            pp = parent[parent]
            if np.array_equal(pp, parent):
                break
            parent = pp
        ea, eb = ea[live], eb[live]


def canonical_from_roots(roots):
    """Rank of each element's root among all roots (graph.py:133-138)."""
    is_root = roots == np.arange(len(roots))
    rank = np.cumsum(is_root) - 1
    return rank[roots], int(is_root.sum())


def _f64_key(x):
    """Order-preserving integer key of a float64 (-0.0 and +0.0 share 0)."""
    bits = struct.unpack("<q", struct.pack("<d", float(x)))[0]
    return bits if bits >= 0 else -(bits & 0x7FFFFFFFFFFFFFFF)


def _f64_from_key(k):
    bits = k if k >= 0 else ((-k) | (1 << 63)) - (1 << 64)
    return struct.unpack("<d", struct.pack("<q", bits))[0]


def dot_cutoff(theta_c):
    """Smallest float64 d with arccos(clip(d, -1, 1)) < theta_c.

    numpy's arccos is monotone non-increasing, so "angle < theta_c" equals
    "dot >= d*" (graph.py:92, 159); found by bisection on the ordered
    integer view of the float64 lattice, using numpy's own arccos.
    """
    theta_c = float(theta_c)

    def kept(d):
        # evaluate through a full SIMD-width vector so numpy takes the same
        # inner loop as for the edge arrays
        v = np.clip(np.full(64, d, np.float64), -1.0, 1.0)
        return bool(np.arccos(v)[17] < theta_c)

    if not kept(1.0):
        return math.inf
    if kept(-1.0):
        return -math.inf
    klo, khi = _f64_key(-1.0), _f64_key(1.0)
    while khi - klo > 1:
        mid = (klo + khi) // 2
        if kept(_f64_from_key(mid)):
            khi = mid
        else:
            klo = mid
    return _f64_from_key(khi)


def components(n64, mask, edges, theta_c):
    """Continuous components (graph.py:141-165).

    Keep an edge iff arccos(clip(n_a . n_b)) < theta_c with the dot summed
    as (x0 + x1) + x2 (numpy's np.sum over a length-3 axis); theta_c=None
    gives one component per valid pixel.  Returns (labels over H*W with -1
    for invalid pixels, component_count).
    """
    flat_mask = mask.ravel()
    verts = np.flatnonzero(flat_mask)
    labels = np.full(flat_mask.size, -1, np.int64)
    if theta_c is None:
        labels[verts] = np.arange(len(verts))
        return labels, len(verts)
    flat = n64.reshape(-1, 3)
    pa = flat[edges[:, 0]] * flat[edges[:, 1]]
    dot = (pa[:, 0] + pa[:, 1]) + pa[:, 2]
    keep = np.arccos(np.clip(dot, -1.0, 1.0)) < float(theta_c)
    compact = np.full(flat_mask.size, -1, np.int64)
    compact[verts] = np.arange(len(verts))
    roots = _union_find_roots(len(verts), compact[edges[keep, 0]], compact[edges[keep, 1]])
    canon, count = canonical_from_roots(roots)
    labels[verts] = canon
    return labels, count


def inter_edge_ids(labels, edges):
    """Edges whose endpoint labels differ (graph.py:186-196)."""
    return np.flatnonzero(labels[edges[:, 0]] != labels[edges[:, 1]])


# -------------------------------------------------------------- continuity


@dataclass
class Coefficients:
    """Per-edge coefficients, indexed like ``edges`` (continuity.py:166-193)."""

    omega_a: np.ndarray
    omega_b: np.ndarray
    gamma_a: np.ndarray
    gamma_b: np.ndarray
    opp_a: np.ndarray
    opp_b: np.ndarray
    valid: np.ndarray


def _reflect(center, other, w, h, flat_mask):
    """Point reflection of ``other`` through ``center`` (continuity.py:196-207)."""
    cu, cv = center % w, center // w
    ru = 2 * cu - other % w
    rv = 2 * cv - other // w
    inside = (ru >= 0) & (ru < w) & (rv >= 0) & (rv < h)
    rid = np.where(inside, rv * w + ru, 0)
    return np.where(inside & flat_mask[rid], rid, -1)


def edge_coefficients(n64, mask, edges, intr, model="milano"):
    """omega / gamma / opposite ids / validity (continuity.py:210-289)."""
    if model not in ("milano", "bini"):
        raise ValueError(f"unknown continuity model {model!r}")
    fx, fy, cx, cy = intr
    h, w = mask.shape
    flat = n64.reshape(-1, 3)
    a, b = edges[:, 0], edges[:, 1]
    na, nb = flat[a], flat[b]
    ua, va = (a % w).astype(np.float64), (a // w).astype(np.float64)
    ub, vb = (b % w).astype(np.float64), (b // w).astype(np.float64)
    ta = rays(fx, fy, cx, cy, ua, va)
    tb = rays(fx, fy, cx, cy, ub, vb)
    if model == "milano":
        tm = rays(fx, fy, cx, cy, 0.5 * (ua + ub), 0.5 * (va + vb))
        p_a = (na * ta).sum(1)
        p_b = (nb * tb).sum(1)
        m_a = (na * tm).sum(1)
        m_b = (nb * tm).sum(1)
        small = np.minimum(np.minimum(np.abs(p_a), np.abs(p_b)),
                           np.minimum(np.abs(m_a), np.abs(m_b)))
        with np.errstate(divide="ignore", invalid="ignore"):
            arg = (m_a * p_b) / (p_a * m_b)
        valid = (small >= EPS_DEN) & (arg > EPS_LOG)
        om = np.zeros(len(a))
        om[valid] = np.log(arg[valid])
        om_a, om_b = om, -om
    else:
        du, dv = ub - ua, vb - va
        horiz = dv == 0
        axis = np.abs(du) + np.abs(dv) == 1
        f_dir = np.where(horiz, fx, fy)
        num_a = np.where(horiz, du * na[:, 0], dv * na[:, 1])
        num_b = np.where(horiz, -du * nb[:, 0], -dv * nb[:, 1])
        den_a = na[:, 0] * (ua - cx) + na[:, 1] * (va - cy) + na[:, 2] * f_dir
        den_b = nb[:, 0] * (ub - cx) + nb[:, 1] * (vb - cy) + nb[:, 2] * f_dir
        valid = axis & (np.abs(den_a) >= EPS_DEN) & (np.abs(den_b) >= EPS_DEN)
        om_a = np.where(valid, num_a / np.where(valid, den_a, 1.0), 0.0)
        om_b = np.where(valid, num_b / np.where(valid, den_b, 1.0), 0.0)
    fm = 0.5 * (fx + fy)
    ga = fm * np.abs((na * (ta / np.linalg.norm(ta, axis=1, keepdims=True))).sum(1))
    gb = fm * np.abs((nb * (tb / np.linalg.norm(tb, axis=1, keepdims=True))).sum(1))
    fm_ = mask.ravel()
    return Coefficients(om_a, om_b, ga, gb, _reflect(a, b, w, h, fm_), _reflect(b, a, w, h, fm_), valid)


def _sigmoid(x):
    """expit restated: 1 / (1 + exp(-x)) (continuity.py:60-62)."""
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def bilateral(co, edges, z, k, sel):
    """Bilateral weights for both directions (continuity.py:292-314)."""
    a, b = edges[sel, 0], edges[sel, 1]

    def side(c, o, opp, g):
        has = opp >= 0
        d_o = z[o] - z[c]
        d_p = np.where(has, z[np.maximum(opp, 0)] - z[c], 0.0)
        s = _sigmoid(k * ((g * g) * (d_p ** 2 - d_o ** 2)))
        return np.where(has, s, 0.5)

    return side(a, b, co.opp_a[sel], co.gamma_a[sel]), side(b, a, co.opp_b[sel], co.gamma_b[sel])


def edge_weights(co, edges, z, k, sel):
    """Total weights valid * gamma^2 * w_bilateral (continuity.py:317-331)."""
    wa, wb = bilateral(co, edges, z, k, sel)
    v = co.valid[sel]
    return (np.where(v, np.square(co.gamma_a[sel]) * wa, 0.0),
            np.where(v, np.square(co.gamma_b[sel]) * wb, 0.0))


def outlier_weight(chi, mode, low, high):
    """Soft / hard / off outlier weights (continuity.py:140-158)."""
    mag = np.abs(np.asarray(chi, np.float64))
    if mode == "off":
        return np.ones_like(mag)
    if mode == "hard":
        return np.where(mag >= high, 0.0, 1.0)
    lt, ut = np.log10(low), np.log10(high)
    x = 2.0 * np.log10(np.maximum(mag, LOG_FLOOR)) - (lt + ut)
    return _sigmoid(1.0 * (4.0 / (lt - ut) * x))


# ------------------------------------------------------------------ solver


def conjugate_gradient(matvec, b, rtol, maxiter):
    """scipy.sparse.linalg.cg restated (scipy 1.18.1): x0 = 0, M = I.

    Returns (x, ok, iterations)."""
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros_like(b), True, 0
    atol = rtol * bn
    x = np.zeros_like(b)
    r = b.copy()
    p = None
    rho_prev = 0.0
    for it in range(maxiter):
        if np.linalg.norm(r) < atol:
            return x, True, it
        rho = float(np.dot(r, r))
        if it == 0:
            p = r.copy()
        else:
            p *= rho / rho_prev
            p += r
        q = matvec(p)
        alpha = rho / float(np.dot(p, q))
        x += alpha * p
        r -= alpha * q
        rho_prev = rho
    return x, False, maxiter


def pair_normal_system(ca, cb, rhs_a, rhs_b, w_a, w_b, n):
    """A^T W A and A^T W b of the interleaved pair rows (solver.py:69-111).

    Row 2i = +x[ca] - x[cb] ~ rhs_a (weight w_a); row 2i+1 = +x[cb] - x[ca] ~
    rhs_b (weight w_b).  A^T W A is the graph Laplacian with edge weight
    w_a + w_b; A^T W b gathers w_a rhs_a - w_b rhs_b at ca and the negation
    at cb.
    """
    c = w_a + w_b
    rows = np.concatenate([ca, cb, ca, cb])
    cols = np.concatenate([cb, ca, ca, cb])
    vals = np.concatenate([-c, -c, c, c])
    mat = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    t = w_a * rhs_a - w_b * rhs_b
    rhs = np.bincount(ca, weights=t, minlength=n) - np.bincount(cb, weights=t, minlength=n)
    return mat, rhs


def fill(labels, count, edges, co, st: Settings, z0=None):
    """Per-component fill from zero log-depth (solver.py:183-239).

    Returns (z_flat, warnings, iterations per component).
    """
    z = np.zeros(labels.size) if z0 is None else z0.copy()
    la = labels[edges[:, 0]]
    intra = np.flatnonzero(la == labels[edges[:, 1]])
    lab_i = la[intra]
    order = np.argsort(lab_i, kind="stable")
    intra = intra[order]
    bounds = np.searchsorted(lab_i[order], np.arange(count + 1))
    valid_ids = np.flatnonzero(labels >= 0)
    lv = labels[valid_ids]
    porder = np.argsort(lv, kind="stable")
    grouped = valid_ids[porder]
    pb = np.searchsorted(lv[porder], np.arange(count + 1))
    sizes = np.diff(pb)
    warnings = []
    iters = np.zeros(count, np.int64)

    def one_pass(zs):
        wa_all, wb_all = edge_weights(co, edges, zs, st.k, intra)
        out = zs.copy()
        for c in range(count):
            if sizes[c] <= 1:
                continue
            pix = grouped[pb[c]:pb[c + 1]]
            e0, e1 = bounds[c], bounds[c + 1]
            eids = intra[e0:e1]
            ca = np.searchsorted(pix, edges[eids, 0])
            cb = np.searchsorted(pix, edges[eids, 1])
            mat, rhs = pair_normal_system(ca, cb, co.omega_a[eids], co.omega_b[eids],
                                          wa_all[e0:e1], wb_all[e0:e1], len(pix))
            if not np.any(rhs):
                x, ok, it = np.zeros(len(pix)), True, 0
            else:
                x, ok, it = conjugate_gradient(mat.dot, rhs, st.cg_tol, max(st.cg_max_iters, len(pix)))
            out[pix] = x
            iters[c] = it
            if not ok:
                warnings.append(f"component {c}: cg hit iteration cap")
        return out

    z = one_pass(z)
    if st.refill_reweighted:
        z = one_pass(z)
    return z, warnings, iters


@dataclass
class ScaleStepResult:
    scales: np.ndarray
    energy: float
    residual: np.ndarray  # (2K,) interleaved rows
    weights: np.ndarray  # (2K,)
    ok: bool


def inter_weights(co, edges, eids, z, t, st: Settings):
    """Directed inter-edge weights for 0-based iteration t (solver.py:253-278)."""
    valid = co.valid[eids]
    if t < st.alignment_iters:
        u = valid.astype(np.float64)
        return u, u.copy()
    wa, wb = edge_weights(co, edges, z, st.k, eids)
    a, b = edges[eids, 0], edges[eids, 1]
    chi_a = z[a] - z[b] - co.omega_a[eids]
    chi_b = z[b] - z[a] - co.omega_b[eids]
    wa = wa * outlier_weight(chi_a, st.reweighting_mode, st.outlier_low, st.outlier_high)
    wb = wb * outlier_weight(chi_b, st.reweighting_mode, st.outlier_low, st.outlier_high)
    return np.where(valid, wa, 0.0), np.where(valid, wb, 0.0)


def project_range(rhs, count, pa, pb, conductance):
    """Remove the roundoff null-space component of A^T W b.

    In exact arithmetic A^T W b sums to zero over every connected part of the
    positive-conductance quotient graph, so this is a no-op; in floating
    point the reference (solver.py:114-121) hands CG a slightly inconsistent
    right-hand side, and when the system is already solved (the second
    alignment iteration, t=1) CG runs to its cap drifting along the constant
    null vector (observed: scales of -5.7e12 and E_1 != E_0 on the golden
    case c5_voronoi48).  Both this oracle and the GPU path subtract the
    per-part mean; DESIGN.md "Reference numerics" documents the deviation.
    """
    live = conductance > 0
    roots = _union_find_roots(count, pa[live], pb[live])
    part, nparts = canonical_from_roots(roots)
    sums = np.bincount(part, weights=rhs, minlength=nparts)
    sizes = np.bincount(part, minlength=nparts)
    return rhs - (sums / sizes)[part]


def scale_step(labels, count, edges, eids, co, z, t, st: Settings):
    """One relative-scale solve (solver.py:153-180, 281-303)."""
    if len(eids) == 0:
        return ScaleStepResult(np.zeros(count), 0.0, np.zeros(0), np.zeros(0), True)
    wa, wb = inter_weights(co, edges, eids, z, t, st)
    a, b = edges[eids, 0], edges[eids, 1]
    pa, pb = labels[a], labels[b]
    ra = co.omega_a[eids] - (z[a] - z[b])
    rb = co.omega_b[eids] - (z[b] - z[a])
    mat, rhs = pair_normal_system(pa, pb, ra, rb, wa, wb, count)
    if not np.any(rhs):
        s, ok = np.zeros(count), True
    else:
        rhs = project_range(rhs, count, pa, pb, wa + wb)
        s, ok, _ = conjugate_gradient(mat.dot, rhs, st.cg_tol, max(st.cg_max_iters, count))
    res = np.empty(2 * len(eids))
    res[0::2] = s[pa] - s[pb] - ra
    res[1::2] = s[pb] - s[pa] - rb
    wts = np.empty(2 * len(eids))
    wts[0::2], wts[1::2] = wa, wb
    return ScaleStepResult(s, float(res @ (wts * res)), res, wts, ok)


def merge(labels, count, pairs, residuals):
    """Union each component with its smallest-residual neighbour
    (graph.py:207-250).  ``pairs`` are the (K, 2) component pairs of the
    inter edges in edge order; ties broken by the smaller edge index."""
    if len(pairs) == 0:
        return labels.copy(), count
    comp = np.concatenate([pairs[:, 0], pairs[:, 1]])
    eidx = np.tile(np.arange(len(pairs)), 2)
    res = np.tile(residuals, 2)
    order = np.lexsort((eidx, res, comp))
    cs = comp[order]
    first = np.searchsorted(cs, np.arange(count), side="left")
    has = (first < len(cs)) & (cs[np.minimum(first, len(cs) - 1)] == np.arange(count))
    sel = np.unique(eidx[order][first[has]])
    roots = _union_find_roots(count, pairs[sel, 0], pairs[sel, 1])
    meta, new_count = canonical_from_roots(roots)
    return np.where(labels >= 0, meta[np.maximum(labels, 0)], -1), new_count


def converged(e_t, e_prev, t, st: Settings):
    """Energy stopping rule (pipeline.py:66-83)."""
    if t >= st.max_iters or e_t <= ENERGY_FLOOR:
        return True
    if t <= st.alignment_iters + 1 or e_prev <= ENERGY_FLOOR:
        return False
    return abs(e_t - e_prev) / e_prev < st.delta_e_max


def digest(z):
    """pipeline.py:58-59."""
    return hashlib.sha256(np.ascontiguousarray(z).tobytes()).hexdigest()[:16]


@dataclass
class OracleResult:
    log_depth: np.ndarray  # (H, W) float64, 0 outside the mask
    filled: np.ndarray  # (H, W)
    labels0: np.ndarray  # (H*W,) int64
    count0: int
    labels: np.ndarray
    count: int
    records: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    iterations: int = 0
    energies: list = field(default_factory=list)
    fill_iters: np.ndarray | None = None
    scales: list = field(default_factory=list)  # per-iteration scale vectors


def run_pipeline(normals, mask, intr, theta_c, st: Settings | None = None,
                 connectivity=8, model="milano", gauge_depth=None) -> OracleResult:
    """Algorithm 1 end to end (pipeline.py:105-248)."""
    st = st or Settings()
    if model == "bini" and connectivity == 8:
        raise ValueError("bini needs connectivity=4")
    n64, m = normalize_normals(normals, mask)
    h, w = m.shape
    records = []
    warnings = []
    t_run = time.perf_counter()
    t0 = time.perf_counter()
    edges, _ = pixel_edges(m, connectivity)
    records.append({"stage": "build_graph", "vertices": int(m.sum()), "edges": len(edges),
                    "wall_ms": (time.perf_counter() - t0) * 1e3})
    t0 = time.perf_counter()
    labels0, count0 = components(n64, m, edges, theta_c)
    records.append({"stage": "form_components", "component_count": count0,
                    "wall_ms": (time.perf_counter() - t0) * 1e3})
    t0 = time.perf_counter()
    co = edge_coefficients(n64, m, edges, intr, model)
    records.append({"stage": "edge_coefficients", "degenerate_edges": int((~co.valid).sum()),
                    "wall_ms": (time.perf_counter() - t0) * 1e3})
    t0 = time.perf_counter()
    z, fw, fit = fill(labels0, count0, edges, co, st)
    warnings.extend(fw)
    records.append({"stage": "fill", "wall_ms": (time.perf_counter() - t0) * 1e3})
    filled = np.where(m.ravel(), z, 0.0).reshape(h, w)

    labels, count = labels0, count0
    eids = inter_edge_ids(labels, edges)
    valid = labels >= 0
    e_prev = ENERGY_FLOOR
    energies = []
    scales = []
    t = 0
    done = False
    while not done:
        ti = time.perf_counter()
        step = scale_step(labels, count, edges, eids, co, z, t, st)
        if not step.ok:
            warnings.append(f"iteration {t}: cg hit iteration cap")
        if count:
            z[valid] += step.scales[labels[valid]]
        scales.append(step.scales)
        t += 1
        extra = {}
        merged = False
        if st.freq_merging is not None and t % st.freq_merging == 0 and count > 1 and len(eids) > 0:
            d_before = digest(z)
            pairs = np.stack([labels[edges[eids, 0]], labels[edges[eids, 1]]], axis=1)
            new_labels, new_count = merge(labels, count, pairs, np.abs(step.residual[0::2]))
            new_eids = inter_edge_ids(new_labels, edges)
            pos = np.searchsorted(eids, new_eids)
            rows = np.empty(2 * len(pos), np.int64)
            rows[0::2], rows[1::2] = 2 * pos, 2 * pos + 1
            r = step.residual[rows]
            e_t = float(r @ (step.weights[rows] * r))
            extra = {"components_before": count, "components_after": new_count,
                     "z_digest_before": d_before, "z_digest_after": digest(z)}
            labels, count, eids = new_labels, new_count, new_eids
            merged = True
        else:
            e_t = step.energy
        done = converged(e_t, e_prev, t, st)
        e_prev = e_t
        energies.append(e_t)
        records.append({"t": t, "E_t": e_t, "component_count": count, "merge_performed": merged,
                        "wall_ms": (time.perf_counter() - ti) * 1e3, **extra})
    target = 0.0 if gauge_depth is None else float(np.log(gauge_depth))
    z += (target - float(np.median(z[valid]))) * valid
    records.append({"stage": "done", "iterations": t, "warnings": len(warnings),
                    "wall_ms": (time.perf_counter() - t_run) * 1e3})
    return OracleResult(np.where(m.ravel(), z, 0.0).reshape(h, w), filled, labels0, count0,
                        labels, count, records, warnings, t, energies, fit, scales)


@dataclass
class BaselineOracleResult:
    log_depth: np.ndarray  # (H, W) float64, 0 outside the mask
    records: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    iterations: int = 0
    energies: list = field(default_factory=list)
    cg_iters: list = field(default_factory=list)


def run_pixel_baseline(normals, mask, intr, st: Settings | None = None, connectivity=8,
                       model="milano", gauge_depth=None) -> BaselineOracleResult:
    """Iteratively reweighted per-pixel integration (pipeline.py:297-369).

    Every outer iteration re-solves the full pixel system (one CG over all
    valid pixels, x0 = 0, pipeline.py:261-285 + solver.py:97-122) with the
    weight schedule of the inter system (solver.py:253-278), and the solution
    replaces z.
    """
    st = st or Settings()
    if model == "bini" and connectivity == 8:
        raise ValueError("bini needs connectivity=4")
    n64, m = normalize_normals(normals, mask)
    h, w = m.shape
    records, warnings, energies, cg_iters = [], [], [], []
    t_run = time.perf_counter()
    edges, _ = pixel_edges(m, connectivity)
    co = edge_coefficients(n64, m, edges, intr, model)
    flat = m.ravel()
    vid = np.flatnonzero(flat)
    compact = np.full(flat.size, -1, np.int64)
    compact[vid] = np.arange(len(vid))
    ca, cb = compact[edges[:, 0]], compact[edges[:, 1]]
    eids = np.arange(len(edges))
    n = len(vid)
    z = np.zeros(flat.size)
    e_prev = ENERGY_FLOOR
    t = 0
    done = False
    while not done:
        ti = time.perf_counter()
        wa, wb = inter_weights(co, edges, eids, z, t, st)
        mat, rhs = pair_normal_system(ca, cb, co.omega_a, co.omega_b, wa, wb, n)
        if n == 0 or len(edges) == 0 or not np.any(rhs):
            x, ok, it = np.zeros(n), True, 0
        else:
            x, ok, it = conjugate_gradient(mat.dot, rhs, st.cg_tol, max(st.cg_max_iters, n))
        if not ok:
            warnings.append(f"iteration {t}: cg hit iteration cap")
        res = np.empty(2 * len(edges))
        res[0::2] = x[ca] - x[cb] - co.omega_a
        res[1::2] = x[cb] - x[ca] - co.omega_b
        wts = np.empty(2 * len(edges))
        wts[0::2], wts[1::2] = wa, wb
        e_t = float(res @ (wts * res))
        z[vid] = x
        cg_iters.append(it)
        t += 1
        done = converged(e_t, e_prev, t, st)
        e_prev = e_t
        energies.append(e_t)
        records.append({"t": t, "E_t": e_t, "component_count": n, "merge_performed": False,
                        "wall_ms": (time.perf_counter() - ti) * 1e3})
    target = 0.0 if gauge_depth is None else float(np.log(gauge_depth))
    z += (target - float(np.median(z[flat]))) * flat
    records.append({"stage": "done", "iterations": t, "warnings": len(warnings),
                    "wall_ms": (time.perf_counter() - t_run) * 1e3})
    return BaselineOracleResult(np.where(flat, z, 0.0).reshape(h, w), records, warnings, t,
                                energies, cg_iters)


# ------------------------------------------------------------------ metrics


def _joint_valid(pred, gt, mask):
    """metrics.py:37-41."""
    ok = np.isfinite(pred) & np.isfinite(gt) & (pred > 0) & (gt > 0)
    if mask is not None:
        ok &= np.asarray(mask, dtype=bool)
    return ok


def evaluate(pred, gt, mask=None):
    """Median-ratio aligned MADE / relative error (metrics.py:44-65).
    Returns (made, relative_error, aligned_scale, valid_pixel_count)."""
    pred = np.asarray(pred, np.float64)
    gt = np.asarray(gt, np.float64)
    ok = _joint_valid(pred, gt, mask)
    if not ok.any():
        raise OracleError("no jointly valid pixel")
    p, g = pred[ok], gt[ok]
    scale = float(np.median(g / p))
    err = np.abs(scale * p - g)
    return float(np.mean(err)), float(np.mean(err / g)), scale, int(ok.sum())


def l1_optimal_scale(pred, gt):
    """Weighted median of gt/pred with weights pred (metrics.py:68-84)."""
    pred = np.asarray(pred, np.float64).ravel()
    gt = np.asarray(gt, np.float64).ravel()
    ratios = gt / pred
    order = np.argsort(ratios, kind="stable")
    cum = np.cumsum(pred[order])
    return float(ratios[order][int(np.searchsorted(cum, 0.5 * cum[-1], side="left"))])


def min_theoretical_made(pred, gt, labels, count, mask=None):
    """Per-component L1-optimal scales, pixel-weighted mean error
    (metrics.py:87-113)."""
    pred = np.asarray(pred, np.float64).ravel()
    gt = np.asarray(gt, np.float64).ravel()
    ok = _joint_valid(pred, gt, None if mask is None else np.asarray(mask).ravel())
    total_err, total_px = 0.0, 0
    for c in range(count):
        pix = np.flatnonzero(labels == c)
        pix = pix[ok[pix]]
        if len(pix) == 0:
            continue
        s = l1_optimal_scale(pred[pix], gt[pix])
        total_err += float(np.sum(np.abs(s * pred[pix] - gt[pix])))
        total_px += len(pix)
    if total_px == 0:
        raise OracleError("no jointly valid pixel in any component")
    return total_err / total_px


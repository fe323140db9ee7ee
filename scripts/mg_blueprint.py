"""Round-2 blueprint: the multigrid-preconditioned fill in the exact data
layout planned for the GPU, in numpy, on one C5 map.

Every level is a list of unknowns keyed (block row, block column, label) and
sorted by that key; each unknown has 8 neighbour indices (same label in the
adjacent block, -1 if absent) and 8 conductances, its diagonal is their sum,
and it has one parent at the next level.  Level 0 is the pixel grid.  Coarse
conductances are fixed-order sums of the finer links between two aggregates
(Galerkin with piecewise-constant prolongation).  The preconditioner is one
V-cycle: damped Jacobi from zero, residual, restriction (sum over children),
recursion, prolongation (add the parent's value), one damped Jacobi sweep; a
fixed number of Jacobi sweeps on the coarsest level.  PCG runs per component
(the hierarchy never mixes labels, so the preconditioner is block-diagonal).

    python scripts/mg_blueprint.py [map index] [coarsest sweeps]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import normint_oracle as O  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

DIRS = [(1, 0), (-1, 1), (0, 1), (1, 1), (-1, 0), (1, -1), (0, -1), (-1, -1)]  # (du, dv)
OPP = [4, 5, 6, 7, 0, 1, 2, 3]


def level0(sc):
    """Pixel-level unknowns of the fill system at z = 0 (oracle.fill)."""
    n64, m = O.normalize_normals(sc.normals.astype(np.float64), sc.mask)
    edges, _ = O.pixel_edges(m, 8)
    labels, count = O.components(n64, m, edges, float(np.deg2rad(3.5)))
    co = O.edge_coefficients(n64, m, edges, sc.intrinsics())
    la = labels[edges[:, 0]]
    intra = np.flatnonzero(la == labels[edges[:, 1]])
    wa, wb = O.edge_weights(co, edges, np.zeros(labels.size), 2.0, intra)
    h, w = m.shape
    sizes = np.bincount(labels[labels >= 0], minlength=count)
    live = (labels >= 0) & (sizes[np.maximum(labels, 0)] > 1)
    pix = np.flatnonzero(live)
    idx = np.full(h * w, -1)
    idx[pix] = np.arange(len(pix))
    nbr = np.full((len(pix), 8), -1)
    cond = np.zeros((len(pix), 8))
    a, b = edges[intra, 0], edges[intra, 1]
    c = wa + wb
    du = (b % w) - (a % w)
    dv = (b // w) - (a // w)
    for d, (ddu, ddv) in enumerate(DIRS[:4]):
        sel = (du == ddu) & (dv == ddv) & (c > 0)
        ia, ib = idx[a[sel]], idx[b[sel]]
        nbr[ia, d], cond[ia, d] = ib, c[sel]
        nbr[ib, OPP[d]], cond[ib, OPP[d]] = ia, c[sel]
    # right-hand side A^T W b (solver.py:83-93)
    t = wa * co.omega_a[intra] - wb * co.omega_b[intra]
    rhs = np.bincount(idx[a], weights=t, minlength=len(pix)) - np.bincount(idx[b], weights=t,
                                                                         minlength=len(pix))
    lev = {"u": pix % w, "v": pix // w, "lab": labels[pix], "nbr": nbr, "cond": cond}
    return lev, rhs, labels[pix]


def coarsen(f, factor=2):
    """(block, label) aggregates of level f, their links and conductances."""
    bu, bv, lab = f["u"] // factor, f["v"] // factor, f["lab"]
    key = (bv.astype(np.int64) << 40) | (bu.astype(np.int64) << 20) | lab
    uniq, parent = np.unique(key, return_inverse=True)
    nc = len(uniq)
    c = {"u": (uniq >> 20) & ((1 << 20) - 1), "v": uniq >> 40, "lab": uniq & ((1 << 20) - 1)}
    nbr = np.full((nc, 8), -1)
    cond = np.zeros((nc, 8))
    pu, pv = c["u"], c["v"]
    for d in range(8):  # fine links leaving the parent block, by the direction of the coarse link
        ok = f["nbr"][:, d] >= 0
        i = np.flatnonzero(ok)
        j = f["nbr"][i, d]
        P, Q = parent[i], parent[j]
        cross = P != Q
        P, Q, cc = P[cross], Q[cross], f["cond"][i[cross], d]
        ddu, ddv = pu[Q] - pu[P], pv[Q] - pv[P]
        for e, (eu, ev) in enumerate(DIRS):
            s2 = (ddu == eu) & (ddv == ev)
            np.add.at(cond[:, e], P[s2], cc[s2])  # fixed order on the GPU: child, direction
            nbr[P[s2], e] = Q[s2]
    c["nbr"], c["cond"] = nbr, cond
    return c, parent


def apply_A(lev, x):
    xn = np.where(lev["nbr"] >= 0, x[np.maximum(lev["nbr"], 0)], 0.0)
    return (lev["cond"] * (x[:, None] - xn)).sum(1)


OVERCORRECT = float(__import__("os").environ.get("MG_OC", "1.0"))  # coarse-correction scale
NU_COARSE = int(__import__("os").environ.get("MG_NU", "1"))  # smoothing sweeps below level 0
NU_FROM = int(__import__("os").environ.get("MG_NU_FROM", "1"))  # ... on levels >= this
GAMMA = int(__import__("os").environ.get("MG_GAMMA", "1"))  # cycle index (2: W-cycle) ...
GAMMA_FROM = int(__import__("os").environ.get("MG_GAMMA_FROM", "1"))  # ... for recursions into levels >= this
GAMMA_TO = int(__import__("os").environ.get("MG_GAMMA_TO", "99"))  # ... and <= this


def vcycle(levels, parents, b, l=0, omega=0.8, coarse_sweeps=20):
    lev = levels[l]
    d = lev["cond"].sum(1)
    dinv = np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 0.0)
    nu = NU_COARSE if l >= NU_FROM else 1
    x = omega * dinv * b
    if l == len(levels) - 1:
        for _ in range(coarse_sweeps - 1):
            x = x + omega * dinv * (b - apply_A(lev, x))
        return x
    for _ in range(nu - 1):
        x = x + omega * dinv * (b - apply_A(lev, x))
    r = b - apply_A(lev, x)
    bc = np.bincount(parents[l], weights=r, minlength=len(levels[l + 1]["lab"]))
    ec = vcycle(levels, parents, bc, l + 1, omega, coarse_sweeps)
    if GAMMA > 1 and GAMMA_FROM <= l + 1 <= GAMMA_TO and l + 1 < len(levels) - 1:
        for _ in range(GAMMA - 1):  # second visit on the coarse residual (symmetric: 2M - MAM)
            ec = ec + vcycle(levels, parents, bc - apply_A(levels[l + 1], ec), l + 1, omega,
                             coarse_sweeps)
    x = x + OVERCORRECT * ec[parents[l]]
    for _ in range(nu):
        x = x + omega * dinv * (b - apply_A(lev, x))
    return x


def pcg_per_component(levels, parents, b, comp, rtol=1e-6, coarse_sweeps=20):
    """One PCG per component, all at once (per-component alpha, beta, stop)."""
    nc = comp.max() + 1
    seg = lambda v: np.bincount(comp, weights=v, minlength=nc)  # noqa: E731
    bn = np.sqrt(seg(b * b))
    x = np.zeros_like(b)
    r = b.copy()
    z = vcycle(levels, parents, r, coarse_sweeps=coarse_sweeps)
    p = z.copy()
    rz = seg(r * z)
    active = bn > 0
    iters = np.zeros(nc, int)
    for it in range(2000):
        rn = np.sqrt(seg(r * r))
        active &= ~(rn < rtol * bn)
        if not active.any():
            break
        iters[active] += 1
        q = apply_A(levels[0], p)
        pq = seg(p * q)
        alpha = np.where(active & (pq > 0), rz / np.where(pq > 0, pq, 1.0), 0.0)
        x += alpha[comp] * p
        r -= alpha[comp] * q
        z = vcycle(levels, parents, r, coarse_sweeps=coarse_sweeps)
        rz_new = seg(r * z)
        beta = np.where(active & (rz > 0), rz_new / np.where(rz > 0, rz, 1.0), 0.0)
        p = np.where(active[comp], z + beta[comp] * p, p)
        rz = rz_new
    return x, iters


if __name__ == "__main__":
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    sc = scenes.config5_map(idx)
    lev0, b, comp_raw = level0(sc)
    _, comp = np.unique(comp_raw, return_inverse=True)
    levels, parents = [lev0], []
    # coarsen until every component is (almost) one aggregate: the coarsest
    # system is then tiny and a few Jacobi sweeps solve it
    first = int(__import__("os").environ.get("MG_FIRST", "2"))
    while len(levels) < 24:
        c, par = coarsen(levels[-1], first if len(levels) == 1 else 2)
        if len(c["lab"]) >= len(levels[-1]["lab"]):
            break
        parents.append(par)
        levels.append(c)
    print("unknowns per level:", [len(l_["lab"]) for l_ in levels])
    x, iters = pcg_per_component(levels, parents, b, comp, coarse_sweeps=sweeps)
    print("MG-PCG iterations per component: max", int(iters.max()), "px-weighted mean",
          round(float((iters[comp]).mean()), 2))
    if __import__("os").environ.get("MG_NOCG"):
        sys.exit(0)
    # the same components with scipy-semantics CG (the current GPU fill)
    cg_it = []
    for c in np.argsort(-np.bincount(comp))[:8]:
        sel = np.flatnonzero(comp == c)
        loc = np.full(len(comp), -1)
        loc[sel] = np.arange(len(sel))
        sub = {"nbr": np.where(levels[0]["nbr"][sel] >= 0, loc[np.maximum(levels[0]["nbr"][sel], 0)], -1),
               "cond": levels[0]["cond"][sel]}
        xc, ok, it = O.conjugate_gradient(lambda v: apply_A(sub, v), b[sel], 1e-6, 5000)
        d = (x[sel] - x[sel].mean()) - (xc - xc.mean())
        cg_it.append((int(c), len(sel), it, int(iters[c]),
                      float(np.linalg.norm(d) / np.linalg.norm(xc - xc.mean()))))
    for c, n, itc, itm, rel in cg_it:
        print(f"component {c}: {n} px, CG {itc} it, blueprint MG-PCG {itm} it, rel diff {rel:.1e}")

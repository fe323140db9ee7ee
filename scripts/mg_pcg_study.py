"""How many iterations would a multigrid-preconditioned fill need?

CPU prototype for the round-2 plan: for the components of a
C5 map, build the fill system exactly as the oracle does (oracle.fill: the
pair normal system A^T W A x = A^T W b at z = 0), then solve it

* with scipy-semantics CG (rtol 1e-6, x0 = 0) -- what the GPU fill does now;
* with CG preconditioned by one V-cycle of an aggregation multigrid whose
  levels are 2x2 pixel blocks *inside the component* (piecewise-constant
  prolongation P, Galerkin coarse operator P^T A P, so coarse conductances
  are sums of fine ones), damped-Jacobi pre/post smoothing, and a direct
  solve on the coarsest level.

Reports per component: size, CG iterations, MG-PCG iterations, and the
relative difference of the two solutions after removing the mean (the
null space).  Work per MG-PCG iteration is about 3-4 fine-level sweeps.

    python scripts/mg_pcg_study.py [map index] [nu (smoothing steps)]
"""
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, ".")
from oracle import normint_oracle as O  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402


def component_systems(sc):
    n64, m = O.normalize_normals(sc.normals.astype(np.float64), sc.mask)
    edges, _ = O.pixel_edges(m, 8)
    labels, count = O.components(n64, m, edges, float(np.deg2rad(3.5)))
    co = O.edge_coefficients(n64, m, edges, sc.intrinsics())
    z = np.zeros(labels.size)
    la = labels[edges[:, 0]]
    intra = np.flatnonzero(la == labels[edges[:, 1]])
    wa, wb = O.edge_weights(co, edges, z, 2.0, intra)
    out = []
    h, w = m.shape
    for c in range(count):
        sel = la[intra] == c
        eids = intra[sel]
        pix = np.flatnonzero(labels == c)
        if len(pix) < 2:
            continue
        ca = np.searchsorted(pix, edges[eids, 0])
        cb = np.searchsorted(pix, edges[eids, 1])
        mat, rhs = O.pair_normal_system(ca, cb, co.omega_a[eids], co.omega_b[eids],
                                        wa[sel], wb[sel], len(pix))
        out.append((c, pix, mat.tocsr(), rhs, w))
    return out


def aggregate(pix_u, pix_v):
    """2x2 block aggregates of a pixel set: (aggregate id per pixel, coarse coords)."""
    bu, bv = pix_u // 2, pix_v // 2
    key = bv.astype(np.int64) * (1 << 20) + bu
    uniq, agg = np.unique(key, return_inverse=True)
    return agg, (uniq % (1 << 20)).astype(np.int64), (uniq >> 20).astype(np.int64)


def hierarchy(A, pu, pv, min_size=400):
    levels = [A]
    Ps = []
    while levels[-1].shape[0] > min_size:
        agg, cu, cv = aggregate(pu, pv)
        n, nc = len(agg), int(agg.max()) + 1
        P = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nc))
        Ac = (P.T @ levels[-1] @ P).tocsr()
        Ps.append(P)
        levels.append(Ac)
        pu, pv = cu, cv
        if nc == n:
            break
    # coarsest: direct solve of the singular (Neumann) system via pinv-free trick:
    # ground one node per connected part is overkill here; use lstsq on dense
    Ad = levels[-1].toarray()
    coarse_pinv = np.linalg.pinv(Ad)
    return levels, Ps, coarse_pinv


def vcycle(levels, Ps, coarse_pinv, b, nu=2, omega=0.8, lvl=0):
    A = levels[lvl]
    if lvl == len(levels) - 1:
        return coarse_pinv @ b
    d = A.diagonal()
    dinv = np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 0.0)
    x = omega * dinv * b
    for _ in range(nu - 1):
        x += omega * dinv * (b - A @ x)
    r = b - A @ x
    P = Ps[lvl]
    x += P @ vcycle(levels, Ps, coarse_pinv, P.T @ r, nu, omega, lvl + 1)
    for _ in range(nu):  # symmetric: same number of post-smoothing steps
        x += omega * dinv * (b - A @ x)
    return x


def pcg(A, b, M, rtol=1e-6, maxiter=5000):
    bn = np.linalg.norm(b)
    x = np.zeros_like(b)
    r = b.copy()
    z = M(r)
    p = z.copy()
    rz = r @ z
    for it in range(maxiter):
        if np.linalg.norm(r) < rtol * bn:
            return x, it
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        z = M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxiter


if __name__ == "__main__":
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    nu = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    sc = scenes.config5_map(idx)
    systems = component_systems(sc)
    tot_cg = tot_mg = 0
    for c, pix, A, b, w in sorted(systems, key=lambda s: -len(s[1]))[:8]:
        if not np.any(b):
            continue
        t0 = time.perf_counter()
        x_cg, ok, it_cg = O.conjugate_gradient(A.dot, b, 1e-6, max(5000, len(pix)))
        t1 = time.perf_counter()
        levels, Ps, cp = hierarchy(A, pix % w, pix // w)
        x_mg, it_mg = pcg(A, b, lambda r: vcycle(levels, Ps, cp, r, nu), 1e-6)
        t2 = time.perf_counter()
        d = (x_mg - x_mg.mean()) - (x_cg - x_cg.mean())
        rel = np.linalg.norm(d) / max(np.linalg.norm(x_cg - x_cg.mean()), 1e-300)
        tot_cg += it_cg * len(pix)
        tot_mg += it_mg * len(pix)
        print(f"component {c}: {len(pix)} px, levels {len(levels)}, CG {it_cg} it ({t1 - t0:.1f} s), "
              f"MG-PCG {it_mg} it ({t2 - t1:.1f} s), rel diff {rel:.2e}", flush=True)
    print(f"px-weighted iterations: CG {tot_cg:.3e}, MG-PCG {tot_mg:.3e} "
          f"(ratio {tot_cg / max(tot_mg, 1):.1f}x)")


def map_level_study(idx=0, nu=1):
    """Label-agnostic variant: one PCG per map over all its components, the
    V-cycle aggregating plain 2x2 pixel blocks of the map grid (blocks on a
    component boundary mix components).  Stop when every component's residual
    is below rtol * its own ||b_c|| (scipy's per-component test)."""
    sc = scenes.config5_map(idx)
    systems = component_systems(sc)
    h, w = sc.mask.shape
    n = h * w
    rows, cols, vals = [], [], []
    b = np.zeros(n)
    comp_of = np.full(n, -1)
    for c, pix, A, bc, _ in systems:
        Ac = A.tocoo()
        rows.append(pix[Ac.row]); cols.append(pix[Ac.col]); vals.append(Ac.data)
        b[pix] = bc
        comp_of[pix] = c
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n))
    act = np.flatnonzero(comp_of >= 0)
    A = A[act][:, act].tocsr()
    b = b[act]
    cid = comp_of[act]
    levels, Ps, cp = hierarchy(A, act % w, act // w)
    bn = np.sqrt(np.bincount(cid, weights=b * b))
    x = np.zeros_like(b)
    r = b.copy()
    z = vcycle(levels, Ps, cp, r, nu)
    p = z.copy()
    rz = r @ z
    for it in range(2000):
        rn = np.sqrt(np.bincount(cid, weights=r * r, minlength=len(bn)))
        if np.all((rn < 1e-6 * bn) | (bn == 0)):
            break
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        z = vcycle(levels, Ps, cp, r, nu)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    print(f"map {idx}: {len(act)} px in {len(systems)} components, label-agnostic 2x2 V-cycle PCG: "
          f"{it} iterations to every component's rtol 1e-6", flush=True)


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "map":
    map_level_study(int(sys.argv[1]), int(sys.argv[2]))


def grid_label_study(idx=0, nu=1, min_cells=64):
    """GPU-friendly component-aware variant: every level is a regular grid
    whose cells carry ONE label -- a 2x2 block takes the label of the most
    pixels of the block (ties: the smallest label) and pixels of any other
    label in the block are left out of the aggregation (they are only
    smoothed).  One PCG per component (the preconditioner is block-diagonal
    by component because aggregates never mix labels)."""
    sc = scenes.config5_map(idx)
    systems = component_systems(sc)
    h, w = sc.mask.shape
    n = h * w
    lab = np.full(n, -1)
    for c, pix, A, bc, _ in systems:
        lab[pix] = c
    # level hierarchy over the grid: label per cell, P maps fine cell -> coarse cell or -1
    levels_lab = [lab.reshape(h, w)]
    while min(levels_lab[-1].shape) > 8 and levels_lab[-1].size > min_cells:
        L = levels_lab[-1]
        hh, ww = (L.shape[0] + 1) // 2, (L.shape[1] + 1) // 2
        Lp = np.full((2 * hh, 2 * ww), -1)
        Lp[:L.shape[0], :L.shape[1]] = L
        blocks = Lp.reshape(hh, 2, ww, 2).transpose(0, 2, 1, 3).reshape(hh, ww, 4)
        coarse = np.full((hh, ww), -1)
        for i in range(4):  # majority label (ties: smallest)
            cand = blocks[..., i]
            cnt = (blocks == cand[..., None]).sum(-1)
            best = (cand >= 0) & ((coarse < 0) | (cnt > (blocks == coarse[..., None]).sum(-1)) |
                                  ((cnt == (blocks == coarse[..., None]).sum(-1)) & (cand < coarse)))
            coarse = np.where(best, cand, coarse)
        levels_lab.append(coarse)
    tot_cg = tot_mg = 0
    for c, pix, A, b, _ in sorted(systems, key=lambda s: -len(s[1]))[:8]:
        if not np.any(b):
            continue
        # per-level membership of component c and the aggregation maps
        Ps = []
        ids = np.full(n, -1)
        ids[pix] = np.arange(len(pix))
        fine_ids, fh, fw = ids.reshape(h, w), h, w
        mats = [A]
        for lv in range(1, len(levels_lab)):
            L = levels_lab[lv]
            ch, cw = L.shape
            cids = np.full((ch, cw), -1)
            mem = L == c
            cids[mem] = np.arange(int(mem.sum()))
            v, u = np.nonzero(fine_ids >= 0)
            src = fine_ids[v, u]
            dst = cids[v // 2, u // 2]
            keep = dst >= 0
            nf, nc = int((fine_ids >= 0).sum()), int(mem.sum())
            if nc == 0:
                break
            P = sp.csr_matrix((np.ones(int(keep.sum())), (src[keep], dst[keep])), shape=(nf, nc))
            Ps.append(P)
            mats.append((P.T @ mats[-1] @ P).tocsr())
            fine_ids = cids
        cp = np.linalg.pinv(mats[-1].toarray())
        x_cg, ok, it_cg = O.conjugate_gradient(A.dot, b, 1e-6, max(5000, len(pix)))
        x_mg, it_mg = pcg(A, b, lambda r: vcycle(mats, Ps, cp, r, nu), 1e-6)
        tot_cg += it_cg * len(pix)
        tot_mg += it_mg * len(pix)
        print(f"component {c}: {len(pix)} px, {len(mats)} levels, CG {it_cg}, grid-label MG-PCG {it_mg}",
              flush=True)
    print(f"grid-label aggregation: px-weighted iterations ratio {tot_cg / max(tot_mg, 1):.1f}x")


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "grid":
    grid_label_study(int(sys.argv[1]), int(sys.argv[2]))

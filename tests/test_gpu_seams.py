"""GPU parity of the reference's seams, called with the
reference's signatures, against the per-seam outputs of the REAL reference
on ``seam_voronoi32`` (tests/golden/make_golden.py:seam_case):

* build_pixel_graph edges, form_components labels, build_quotient edge ids,
  merge_components labels: bit-exact;
* build_edge_coefficients omega / gamma / valid / opp: omega and gamma to
  1e-12 relative (both are float64 transcendental chains), the rest exact;
* fill_components: within 2e-5 (fp32 multigrid PCG vs scipy's fp64 CG);
* relative_scale_step at t = 0 and t = 2: scales within the north-star
  tolerance (1e-4 relative / 1e-3 px), weights to 1e-9, energy to 1e-6.

Plus reference-typed inputs: objects shaped like ``normint.NormalMap``,
``CameraIntrinsics``, ``SolveSettings`` and ``WeightParams`` go straight into
``run_pipeline``.
"""

import os
from dataclasses import dataclass

import numpy as np
import pytest

from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_11508_b200 as nb  # noqa: E402
from oracle import normint_oracle as O  # noqa: E402

THETA = float(np.deg2rad(3.5))


@pytest.fixture(scope="module")
def seam():
    d = dict(np.load(os.path.join(GOLDEN, "seam_voronoi32.npz")))
    # the reference renormalised these float64 normals (NormalMap.create)
    nm = nb.NormalMap.create(d["normals"].astype(np.float64), d["mask"])
    intr = nb.CameraIntrinsics(*d["intr"])
    g = nb.build_pixel_graph(nm, 8)
    p = nb.form_components(g, nm, THETA)
    co = nb.build_edge_coefficients(nm, g, intr, "milano")
    return d, nm, intr, g, p, co


def test_graph_and_components(seam):
    d, nm, intr, g, p, co = seam
    assert np.array_equal(g.edges, d["edges"].astype(np.int64))
    assert g.edge_count == len(d["edges"]) and g.vertex_count == int(d["mask"].sum())
    assert p.component_count == int(d["count0"])
    assert np.array_equal(p.labels, d["labels0"].astype(np.int64))


def test_edge_coefficients(seam):
    d, nm, intr, g, p, co = seam
    assert np.array_equal(co.edges, d["edges"])
    assert np.array_equal(co.valid, d["valid"])
    assert np.array_equal(co.opp_a, d["opp_a"]) and np.array_equal(co.opp_b, d["opp_b"])
    for ours, ref in ((co.omega_to_a, "omega_a"), (co.omega_to_b, "omega_b"),
                      (co.gamma_a, "gamma_a"), (co.gamma_b, "gamma_b")):
        np.testing.assert_allclose(ours, d[ref], rtol=1e-12, atol=1e-15, err_msg=ref)
    assert np.array_equal(co.omega_to_b, -co.omega_to_a)  # exact antisymmetry (Milano)


def test_fill_quotient_scale_merge(seam):
    d, nm, intr, g, p, co = seam
    st = nb.SolveSettings(worker_count=1)
    wp = nb.WeightParams()
    z, warns = nb.fill_components(p, g, co, wp, st)
    assert warns == []
    assert np.abs(z - d["filled"])[d["mask"].ravel()].max() < 2e-5
    q = nb.build_quotient(g, p)
    assert np.array_equal(q.edge_ids, d["inter_edge_ids"].astype(np.int64))
    assert np.array_equal(q.inter_edges, d["edges"][d["inter_edge_ids"]].astype(np.int64))
    lab = d["labels0"].astype(np.int64)
    assert np.array_equal(q.comp_pairs, lab[q.inter_edges])
    zc = d["filled"].copy()  # continue from the reference's own fill, as it did
    steps = {}
    for t in (0, 2):
        s = nb.relative_scale_step(q, p, zc, t, st, wp, co)
        steps[t] = s
        assert s.cg_converged
        sref = d[f"scales_t{t}"]
        # scales are a gauge-free difference: compare them centred
        err = np.abs((s.scales - s.scales.mean()) - (sref - sref.mean()))
        assert err.max() <= 1e-4 * max(np.abs(sref).max(), 1.0) + 1e-3 / float(d["intr"][0])
        np.testing.assert_allclose(s.weights, d[f"weights_t{t}"], rtol=1e-9, atol=1e-12)
        assert abs(s.energy - float(d[f"energy_t{t}"])) <= 1e-6 * float(d[f"energy_t{t}"]) + 1e-18
        lv = lab >= 0
        zc[lv] += d[f"scales_t{t}"][lab[lv]]
    np.testing.assert_allclose(steps[2].residual, d["residual_t2"], rtol=1e-6, atol=1e-9)
    merged = nb.merge_components(q, p, np.abs(d["residual_t2"][0::2]))
    assert merged.component_count == int(d["merged_count"])
    assert merged.version == p.version + 1
    assert np.array_equal(merged.labels, d["merged_labels"].astype(np.int64))
    # merging is pure relabelling: p itself is untouched
    assert np.array_equal(p.labels, lab)


def test_seams_accept_reference_partition(seam):
    d, nm, intr, g, p, co = seam

    @dataclass(frozen=True)
    class RefPartition:  # normint.graph.Partition's fields (graph.py:101-112)
        labels: np.ndarray
        component_count: int
        version: int = 0

    rp = RefPartition(d["labels0"].astype(np.int64), int(d["count0"]))
    q = nb.build_quotient(g, rp)
    assert np.array_equal(q.edge_ids, d["inter_edge_ids"].astype(np.int64))
    merged = nb.merge_components(q, rp, np.abs(d["residual_t2"][0::2]))
    assert np.array_equal(merged.labels, d["merged_labels"].astype(np.int64))


def test_run_pipeline_takes_reference_objects():
    """Objects with the reference's fields (geometry.py:31-113, solver.py:26,
    continuity.py:42) go into run_pipeline unchanged; the result equals the
    one from this package's own types."""
    from paper_2510_11508_b200 import scenes

    @dataclass(frozen=True)
    class RefNormalMap:
        normals: np.ndarray
        mask: np.ndarray

    @dataclass(frozen=True)
    class RefIntrinsics:
        fx: float
        fy: float
        cx: float
        cy: float

    @dataclass(frozen=True)
    class RefSettings:
        cg_tol: float = 1e-6
        cg_max_iters: int = 5000
        delta_e_max: float = 1e-3
        max_iters: int = 150
        alignment_iters: int = 2
        freq_merging: int | None = 3
        worker_count: int = 4
        refill_reweighted: bool = False

    @dataclass(frozen=True)
    class RefWeights:
        k: float = 2.0
        outlier_low: float = 1e-5
        outlier_high: float = 1e-3
        reweighting_mode: str = "hard"

    sc = scenes.config4(3, size=64, cells=8)
    ours = nb.NormalMap.create(sc.normals, sc.mask)
    # what normint.NormalMap.create holds: float64, renormalised
    ref_nm = RefNormalMap(np.array(ours.normals), np.array(ours.mask))
    r_ref = nb.run_pipeline(ref_nm, RefIntrinsics(*sc.intrinsics()), THETA, RefSettings(),
                            RefWeights())
    r_own = nb.run_pipeline(ours, nb.CameraIntrinsics(*sc.intrinsics()), THETA,
                            nb.SolveSettings(freq_merging=3),
                            nb.WeightParams(reweighting_mode="hard"))
    assert np.array_equal(r_ref.partition0.labels, r_own.partition0.labels)
    assert r_ref.iterations == r_own.iterations
    assert np.array_equal(r_ref.log_depth.values, r_own.log_depth.values)
    # and against the oracle on the same float64 normals
    o = O.run_pipeline(np.array(ours.normals), sc.mask, sc.intrinsics(), THETA,
                       O.Settings(freq_merging=3, reweighting_mode="hard"))
    assert np.array_equal(r_ref.partition0.labels, o.labels0)

"""GPU parity: the CUDA path (through the C ABI) against the golden fixtures
produced by the reference and against the CPU oracle on the same inputs.

Bars (BASELINE.json north star):
* component labels bit-exact (canonical: rank of smallest pixel id);
* depth after the reference's own median gauge within
  mean|d_gpu - d_ref| <= 1e-4 * mean|d_ref| + 1e-3 px  (tests/parity.py);
* per-component scales (final z - filled z) within the same tolerance.
"""

import glob
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN, golden_cases
from tests.parity import assert_depth_close, depth_error

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402
from oracle import normint_oracle as O  # noqa: E402

PIPE_CASES = golden_cases()
BASELINE_CASES = golden_cases("pb_")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def opts_of(d):
    return json.loads(str(d["options"]))


def run_gpu(normals, mask, intr, opts):
    theta = opts.get("theta_c_deg", 3.5)
    nm = nb.NormalMap.create(normals, mask)
    st = nb.SolveSettings(freq_merging=opts.get("merge_freq"),
                          refill_reweighted=bool(opts.get("refill", False)))
    wp = nb.WeightParams(reweighting_mode=opts.get("reweighting", "soft"))
    return nb.run_pipeline(nm, nb.CameraIntrinsics(*intr),
                           None if theta is None else float(np.deg2rad(theta)), st, wp,
                           opts.get("connectivity", 8), opts.get("model", "milano"),
                           opts.get("gauge_depth"))


def reference_drifted(d):
    text = json.loads(str(d["warning_text"])) if "warning_text" in d else []
    return any(w.startswith("iteration") for w in text)


@pytest.mark.parametrize("name", PIPE_CASES)
def test_labels_bit_exact_vs_reference(name):
    d = load(name)
    r = run_gpu(d["normals"], d["mask"], tuple(d["intr"]), opts_of(d))
    assert r.partition0.component_count == int(d["count0"])
    assert np.array_equal(r.partition0.labels, d["labels0"].astype(np.int64))


@pytest.mark.parametrize("name", PIPE_CASES)
def test_pipeline_vs_reference(name):
    d = load(name)
    mask = d["mask"]
    r = run_gpu(d["normals"], mask, tuple(d["intr"]), opts_of(d))
    fx = float(d["intr"][0])
    # fill: the per-component solution (fp32 CG vs scipy fp64 CG)
    fill_err = np.abs(r.filled.values - d["filled"])[mask]
    assert fill_err.max() < 2e-5, fill_err.max()
    if reference_drifted(d):
        # The reference's own scale CG hit its cap here: its trajectory is
        # driven by roundoff in the singular scale system (DESIGN.md,
        # "Reference numerics"; oracle.project_range), so iterations and
        # energies are not comparable and test_pipeline_vs_oracle holds the
        # exact bar.  Against the drifted reference: the same initial
        # partition and a depth divergence that stays bounded (measured
        # 1.36e-3 = 13x the north-star bound on c5_voronoi48; asserted <= 20x).
        # After the capped iteration the two trajectories reweight different
        # iterates and settle on different energies (0.215 vs 0.170), so
        # energies are not compared.
        assert np.array_equal(r.partition0.labels, d["labels0"].astype(np.int64))
        err, bound = depth_error(r.log_depth.values, d["log_depth"], mask, fx)
        print(f"{name}: drifted reference, depth error {err:.3e} (bound {bound:.3e})")
        assert err <= 20 * bound, (err, bound)
        return
    assert r.iterations == int(d["iterations"])
    assert r.partition.component_count == int(d["count"])
    assert np.array_equal(r.partition.labels, d["labels"].astype(np.int64))
    assert_depth_close(r.log_depth.values, d["log_depth"], mask, fx)
    if r.iterations < 150:
        np.testing.assert_allclose(r.energies, d["energies"], rtol=2e-3, atol=1e-9)
    else:  # oscillating run (c1_hemi64): only the leading energies are comparable
        np.testing.assert_allclose(r.energies[:4], d["energies"][:4], rtol=2e-3, atol=1e-9)
    rec = json.loads(str(d["records"]))
    assert [x.get("stage") for x in r.records] == [x.get("stage") for x in rec]
    for a, b in zip(r.records, rec):
        assert set(a) == set(b) | {"wall_ms"}
        for k in ("vertices", "edges", "component_count", "degenerate_edges", "t",
                  "merge_performed", "components_before", "components_after", "iterations"):
            if k in b:
                assert a[k] == b[k], (k, a[k], b[k])


@pytest.mark.parametrize("name", PIPE_CASES)
def test_pipeline_vs_oracle(name):
    d = load(name)
    mask = d["mask"]
    o = opts_of(d)
    r = run_gpu(d["normals"], mask, tuple(d["intr"]), o)
    theta = o.get("theta_c_deg", 3.5)
    ref = O.run_pipeline(d["normals"].astype(np.float64), mask, tuple(d["intr"]),
                         None if theta is None else float(np.deg2rad(theta)),
                         O.Settings(freq_merging=o.get("merge_freq"),
                                    reweighting_mode=o.get("reweighting", "soft"),
                                    refill_reweighted=bool(o.get("refill", False))),
                         o.get("connectivity", 8), o.get("model", "milano"), o.get("gauge_depth"))
    assert np.array_equal(r.partition0.labels, ref.labels0)
    if ref.iterations < 150:
        assert r.iterations == ref.iterations
        assert np.array_equal(r.partition.labels, ref.labels)
    assert_depth_close(r.log_depth.values, ref.log_depth, mask, float(d["intr"][0]))


def test_deterministic_reruns():
    sc = scenes.config4(3, size=96, cells=14)
    a = run_gpu(sc.normals, sc.mask, sc.intrinsics(), {"merge_freq": 5})
    b = run_gpu(sc.normals, sc.mask, sc.intrinsics(), {"merge_freq": 5})
    assert np.array_equal(a.log_depth.values, b.log_depth.values)
    assert np.array_equal(a.filled.values, b.filled.values)
    assert a.energies == b.energies

    def strip(rs):
        return [{k: v for k, v in x.items() if k != "wall_ms"} for x in rs]

    assert strip(a.records) == strip(b.records)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_full_size_configs_vs_oracle(cfg):
    sc = scenes.CONFIGS[cfg]()
    theta = float(np.deg2rad(3.5))
    nm = nb.NormalMap.create(sc.normals, sc.mask)
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), theta)
    ref = O.run_pipeline(sc.normals.astype(np.float64), sc.mask, sc.intrinsics(), theta)
    assert np.array_equal(r.partition0.labels, ref.labels0)
    err, bound = depth_error(r.log_depth.values, ref.log_depth, sc.mask, sc.fx)
    print(f"{cfg}: iters gpu={r.iterations} oracle={ref.iterations} depth err {err:.3e} bound {bound:.3e}")
    assert err <= bound


def test_batch_equals_single_maps():
    maps = [scenes.config5_map(i, size=64, cells=5) for i in range(3)]
    nms = [nb.NormalMap.create(m.normals, m.mask) for m in maps]
    intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
    theta = float(np.deg2rad(3.5))
    batch = nb.run_pipeline_batch(nb.stack(nms), intr, theta)
    for i, m in enumerate(maps):
        single = nb.run_pipeline(nms[i], intr[i], theta)
        assert np.array_equal(batch[i].partition0.labels, single.partition0.labels)
        assert batch[i].iterations == single.iterations
        assert_depth_close(batch[i].log_depth.values, single.log_depth.values, m.mask, m.fx)


def test_errors_like_reference():
    n = np.zeros((4, 4, 3), np.float32)
    n[..., 2] = -1
    with pytest.raises(nb.EmptyMask):
        nm = nb.NormalMap.create(n, np.zeros((4, 4), bool))
        nb.run_pipeline(nm, nb.CameraIntrinsics(1, 1, 0, 0), 0.1)
    bad = n.copy()
    bad[1, 1, 2] = -1.01
    with pytest.raises(ValueError):
        nb.NormalMap.create(bad)
    nm = nb.NormalMap.create(n)
    with pytest.raises(ValueError):
        nb.run_pipeline(nm, nb.CameraIntrinsics(1, 1, 0, 0), 0.1, connectivity=8, model="bini")


# ------------------------------------------------------- pixel-level baseline


def run_gpu_baseline(d):
    o = opts_of(d)
    nm = nb.NormalMap.create(d["normals"], d["mask"])
    return nb.run_pixel_baseline(nm, nb.CameraIntrinsics(*tuple(d["intr"])), nb.SolveSettings(),
                                 nb.WeightParams(reweighting_mode=o.get("reweighting", "soft")),
                                 o.get("connectivity", 8), o.get("model", "milano"),
                                 o.get("gauge_depth"))


@pytest.mark.parametrize("name", BASELINE_CASES)
def test_pixel_baseline_vs_reference(name):
    """run_pixel_baseline (pipeline.py:297-369) on the GPU: same outer
    iterations, records and warnings as the reference, depth within the
    north-star tolerance, energies to the fp32-CG precision."""
    d = load(name)
    mask = d["mask"]
    r = run_gpu_baseline(d)
    assert r.iterations == int(d["iterations"])
    assert len(r.warnings) == int(d["warnings"])
    assert_depth_close(r.log_depth.values, d["log_depth"], mask, float(d["intr"][0]))
    np.testing.assert_allclose(r.energies, d["energies"], rtol=2e-3, atol=1e-9)
    rec = json.loads(str(d["records"]))
    assert [x.get("stage") for x in r.records] == [x.get("stage") for x in rec]
    for a, b in zip(r.records, rec):
        assert set(a) == set(b) | {"wall_ms"}
        for k in ("t", "component_count", "merge_performed", "iterations", "warnings"):
            if k in b:
                assert a[k] == b[k], (k, a[k], b[k])


def test_pixel_baseline_batch_equals_single_maps():
    cases = [load(n) for n in ("pb_voronoi40", "pb_hemi40")]
    # same size maps only: pad the hemisphere case's mask/normals are 40x40 too
    normals = np.stack([c["normals"] for c in cases])
    masks = np.stack([c["mask"] for c in cases])
    nm = nb.NormalMap.create(normals, masks)
    res = nb.run_pixel_baseline_batch(nm, [nb.CameraIntrinsics(*tuple(c["intr"])) for c in cases])
    for c, rb in zip(cases, res):
        rs = run_gpu_baseline(c)
        assert rb.iterations == rs.iterations
        assert np.array_equal(rb.log_depth.values, rs.log_depth.values)
        assert rb.energies == rs.energies


def test_refill_changes_the_fill():
    """solver.py:237-238: the second pass uses bilateral weights at the filled
    state (reference test_solver.py:218-231)."""
    d = load("refill_voronoi48")
    o = opts_of(d)
    a = run_gpu(d["normals"], d["mask"], tuple(d["intr"]), {k: v for k, v in o.items() if k != "refill"})
    b = run_gpu(d["normals"], d["mask"], tuple(d["intr"]), o)
    assert not np.array_equal(a.filled.values, b.filled.values)
    err = np.abs(b.filled.values - d["filled"])[d["mask"]]
    assert err.max() < 2e-5, err.max()



# ------------------------------------------------------------------- metrics


@pytest.mark.parametrize("name", golden_cases("metrics_"))
def test_gpu_metrics_match_reference(name):
    """ni_evaluate / ni_min_theoretical_made vs the reference's metrics.py:
    the aligned scale (an exact median) and the count bit-exact, the sums to
    summation-order precision."""
    from paper_2510_11508_b200 import metrics

    d = load(name)
    rep = metrics.evaluate(d["pred"], d["gt"], d["mask"])
    assert rep.valid_pixel_count == int(d["valid_pixel_count"])
    assert rep.aligned_scale == float(d["aligned_scale"])
    assert np.isclose(rep.made, float(d["made"]), rtol=1e-12)
    assert np.isclose(rep.relative_error, float(d["relative_error"]), rtol=1e-12)

    class P:  # a reference-style partition of this map
        labels = d["labels"]
        component_count = int(d["ncomp"])

    mtm = metrics.min_theoretical_made(d["pred"], d["gt"], P, d["mask"])
    assert np.isclose(mtm, float(d["min_theoretical_made"]), rtol=1e-12)
    ok = np.isfinite(d["pred"]) & (d["pred"] > 0) & d["mask"]
    assert metrics.l1_optimal_scale(d["pred"][ok][:500], d["gt"][ok][:500]) == float(d["l1_scale"])


def test_gpu_metrics_batch_equals_single():
    from paper_2510_11508_b200 import metrics

    a, b = load("metrics_c"), load("metrics_c")
    b = {k: v for k, v in b.items()}
    b["pred"] = b["pred"] * 1.7
    reps = metrics.evaluate_batch(np.stack([a["pred"], b["pred"]]), np.stack([a["gt"], b["gt"]]),
                                  np.stack([a["mask"], b["mask"]]))
    assert reps[0] == metrics.evaluate(a["pred"], a["gt"], a["mask"])
    assert reps[1] == metrics.evaluate(b["pred"], b["gt"], b["mask"])


def test_merge_events_preserve_depth():
    """Reference test_pipeline.py:44-57 on the GPU path: merges relabel only,
    so the z digests before and after a merge agree."""
    d = load("bump_ref_merge")
    r = run_gpu(d["normals"], d["mask"], tuple(d["intr"]), opts_of(d))
    merges = [x for x in r.records if x.get("merge_performed")]
    assert merges
    for rec in merges:
        assert isinstance(rec["z_digest_before"], str) and len(rec["z_digest_before"]) == 16
        assert rec["z_digest_before"] == rec["z_digest_after"]
        assert rec["components_after"] < rec["components_before"]
    assert r.partition.component_count < r.partition0.component_count


# ------------------------------------------- BASELINE sizes (C3, one C5 map)


def test_full_size_c5_map_vs_oracle():
    """One BASELINE C5 map (1024^2, 1 M valid px) end to end: labels bit-exact,
    same outer iterations, filled state and depth within the north-star
    tolerance of the float64 oracle.  (The float64 residual of an fp32 iterate
    is bounded by cond(A) * eps32, ~3e-3 here, so the solution, not the
    residual, is what is compared.)"""
    sc = scenes.config5_map(0)
    theta = float(np.deg2rad(3.5))
    nm = nb.NormalMap.create(sc.normals, sc.mask)
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), theta)
    ref = O.run_pipeline(sc.normals.astype(np.float64), sc.mask, sc.intrinsics(), theta)
    assert np.array_equal(r.partition0.labels, ref.labels0)
    assert r.iterations == ref.iterations
    assert_depth_close(r.log_depth.values, ref.log_depth, sc.mask, sc.fx)
    fill_err = np.abs(r.filled.values - ref.filled)[sc.mask]
    assert fill_err.max() < 2e-5, fill_err.max()
    assert_depth_close(r.filled.values, ref.filled, sc.mask, sc.fx, what="filled")


@pytest.mark.slow
def test_full_size_c3_vs_oracle():
    """BASELINE C3 (2048^2, 3.0 M valid px) against the oracle (~90 s of CPU)."""
    sc = scenes.CONFIGS["C3"]()
    theta = float(np.deg2rad(3.5))
    nm = nb.NormalMap.create(sc.normals, sc.mask)
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), theta)
    ref = O.run_pipeline(sc.normals.astype(np.float64), sc.mask, sc.intrinsics(), theta)
    assert np.array_equal(r.partition0.labels, ref.labels0)
    assert r.iterations == ref.iterations
    assert_depth_close(r.log_depth.values, ref.log_depth, sc.mask, sc.fx)

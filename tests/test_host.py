"""CPU tests of the host side: the C-ABI library loads and exports every
symbol include/normint_b200.h declares (no compute without a GPU), the
threshold and settings logic mirrors the reference, and the product package
never touches the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "normint_b200.h")


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\**\s*(ni_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_11508_b200 import _lib, build

    build.build()
    return _lib.load()


def test_header_declares_the_abi():
    names = header_functions()
    for required in ("ni_normalize", "ni_components", "ni_coefficients", "ni_fill",
                     "ni_inter_edges", "ni_quotient_build", "ni_scale_step", "ni_merge",
                     "ni_gauge", "ni_last_error", "ni_version"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2510_11508_b200 import _lib

    for name in header_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes signatures"


def test_host_only_entry_points(lib):
    from paper_2510_11508_b200 import _lib

    assert b"sm_100a" in lib.ni_version()
    assert _lib.size_query(lib.ni_components_workspace_size, 1, 64, 64) > 64 * 64 * 12
    assert _lib.size_query(lib.ni_fill_workspace_size, 2, 64, 64, 8, 10, 0) > 2 * 64 * 64 * 20
    assert (_lib.size_query(lib.ni_fill_workspace_size, 2, 64, 64, 8, 10, 1)
            > _lib.size_query(lib.ni_fill_workspace_size, 2, 64, 64, 8, 10, 0))
    assert _lib.size_query(lib.ni_pair_energy_workspace_size, 3) > 0
    assert _lib.size_query(lib.ni_inter_edges_workspace_size, 1, 32, 32, 4) > 0
    assert _lib.size_query(lib.ni_keys_filter_workspace_size, 100) > 0
    assert _lib.size_query(lib.ni_quotient_workspace_size, 100, 10, 2) > 0
    assert _lib.size_query(lib.ni_scale_step_workspace_size, 100, 10, 2) > 0
    assert _lib.size_query(lib.ni_merge_workspace_size, 100, 10, 2) > 0
    assert _lib.size_query(lib.ni_gauge_workspace_size, 3, 16, 16) > 0
    # argument validation happens before any device work
    st = lib.ni_coefficients(None, None, None, 1, 4, 4, 8, 1, None, None, None, None, None, None,
                             None)
    assert st == _lib.NI_ERR_INVALID_ARG
    assert "connectivity=4" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(st, "x")


def test_dot_cutoff_matches_oracle():
    from oracle import normint_oracle as O
    from paper_2510_11508_b200 import dot_cutoff

    for deg in (0.5, 2.0, 3.5, 5.0, 30.0, 179.0):
        th = float(np.deg2rad(deg))
        assert dot_cutoff(th) == O.dot_cutoff(th)
    assert dot_cutoff(0.0) == float("inf")  # nothing is strictly below 0


def test_settings_validation_mirrors_reference():
    from paper_2510_11508_b200 import SolveSettings, WeightParams

    for kw in ({"cg_tol": 0}, {"max_iters": 0}, {"alignment_iters": -1}, {"freq_merging": 0},
               {"worker_count": 0}):
        with pytest.raises(ValueError):
            SolveSettings(**kw)
    for kw in ({"k": 0}, {"outlier_low": 1e-3, "outlier_high": 1e-5}, {"reweighting_mode": "x"}):
        with pytest.raises(ValueError):
            WeightParams(**kw)
    assert WeightParams(reweighting_mode="hard").mode_code == 2


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_11508_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2510_11508_b200 as nb

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        nb.NormalMap.create(np.zeros((4, 4, 3), np.float32))


def test_bench_reference_arm_line():
    """bench.py --impl reference (the driver's reference arm) runs on the host
    cores without a GPU and prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1


def test_cli_flags_map_to_settings_like_the_reference():
    """RunConfig mapping of `integrate` (cli.py:28-75, 104-128), no GPU needed."""
    from paper_2510_11508_b200 import cli

    ap = cli.build_parser()
    a = ap.parse_args(["integrate", "--normals", "n.pfm", "--intrinsics", "i.json", "--output",
                       "o.pfm", "--theta-c", "none", "--merge-freq", "4", "--reweighting", "hard",
                       "--k", "3", "--max-iters", "9", "--alignment-iters", "1",
                       "--delta-e-max", "1e-4", "--connectivity", "4",
                       "--continuity-model", "bini", "--workers", "2"])
    cfg = cli.RunConfig.from_args(a)
    assert cfg.theta_c is None and cfg.connectivity == 4 and cfg.continuity_model == "bini"
    st, wp = cfg.solve_settings(), cfg.weight_params()
    assert (st.freq_merging, st.max_iters, st.alignment_iters, st.delta_e_max, st.worker_count) \
        == (4, 9, 1, 1e-4, 2)
    assert (wp.reweighting_mode, wp.k) == ("hard", 3.0)
    d = cli.RunConfig.from_args(ap.parse_args(["integrate", "--normals", "n", "--intrinsics", "i",
                                               "--output", "o", "--merge-freq", "off"]))
    assert d.merge_freq is None and abs(d.theta_c - np.deg2rad(3.5)) == 0
    assert cli.main(["integrate", "--normals", "n"]) == 2  # usage error
    assert cli.main(["integrate", "--normals", "n", "--intrinsics", "i", "--output", "o",
                     "--merge-freq", "0"]) == 2


def test_reference_settings_objects_are_coerced():
    from dataclasses import dataclass

    from paper_2510_11508_b200.geometry import as_intrinsics
    from paper_2510_11508_b200.settings import as_settings, as_weights

    @dataclass(frozen=True)
    class RefSettings:  # normint.solver.SolveSettings fields
        cg_tol: float = 1e-7
        cg_max_iters: int = 100
        delta_e_max: float = 1e-3
        max_iters: int = 7
        alignment_iters: int = 2
        freq_merging: int | None = 2
        worker_count: int = 1
        refill_reweighted: bool = True

    st = as_settings(RefSettings())
    assert (st.cg_tol, st.cg_max_iters, st.max_iters, st.freq_merging, st.refill_reweighted) == \
        (1e-7, 100, 7, 2, True)

    class W:
        k, outlier_low, outlier_high, reweighting_mode = 1.5, 1e-6, 1e-2, "off"

    assert as_weights(W()).mode_code == 0 and as_weights(None) is None

    class I:
        fx, fy, cx, cy = 10.0, 11.0, 3.0, 4.0

    assert as_intrinsics(I()).as_tuple() == (10.0, 11.0, 3.0, 4.0)
    try:
        import normint  # the real reference, when importable (build container)
    except ImportError:
        return
    ref = normint.SolveSettings(freq_merging=3)
    assert as_settings(ref).freq_merging == 3
    assert as_intrinsics(normint.CameraIntrinsics(5.0, 5.0, 1.0, 2.0)).cx == 1.0

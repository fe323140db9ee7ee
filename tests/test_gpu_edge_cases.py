"""GPU known-answer and edge-case tests: the reference's own small exact
cases mirrored on the CUDA path, ragged and degenerate
shapes the strip decomposition of the fill must handle (maps narrower or
shorter than one 30 x 30 strip, widths that are not a multiple of 30, holes,
isolated pixels), and the scheduler under its non-default claim patterns.

Every case runs the CUDA path through the C ABI and the CPU oracle on the
same inputs: labels bit-exact, same outer iterations and merged partition,
depth within the north-star tolerance (tests/parity.py).
"""

import os

import numpy as np
import pytest

from tests.parity import assert_depth_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402
from oracle import normint_oracle as O  # noqa: E402


def _tilted(deg, azimuth=0.0):
    t, a = np.deg2rad(deg), np.deg2rad(azimuth)
    return np.array([np.sin(t) * np.cos(a), np.sin(t) * np.sin(a), -np.cos(t)])


def run_both(normals, mask, intr, theta_deg=3.5, connectivity=8, model="milano",
             merge_freq=None):
    """GPU and oracle on identical fp32 normals; returns (gpu, oracle)."""
    normals = np.ascontiguousarray(normals, np.float32)
    mask = np.ascontiguousarray(mask, bool)
    theta = None if theta_deg is None else float(np.deg2rad(theta_deg))
    nm = nb.NormalMap.create(normals, mask)
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*intr), theta,
                        nb.SolveSettings(freq_merging=merge_freq), None, connectivity, model)
    ref = O.run_pipeline(normals.astype(np.float64), mask, intr, theta,
                         O.Settings(freq_merging=merge_freq), connectivity, model)
    return r, ref


def assert_parity(r, ref, mask, intr):
    assert np.array_equal(r.partition0.labels, ref.labels0)
    assert r.partition0.component_count == ref.count0
    assert r.iterations == ref.iterations
    assert np.array_equal(r.partition.labels, ref.labels)
    assert_depth_close(r.log_depth.values, ref.log_depth, mask, float(intr[0]))


def test_two_halves_two_components():
    """test_graph.py:153-166: a 4x4 map whose halves differ by 10 degrees at
    theta_c = 5 degrees -> 2 components, the first pixel's labelled 0."""
    n = np.zeros((4, 4, 3))
    n[:, :2] = _tilted(0.0)
    n[:, 2:] = _tilted(10.0)
    mask = np.ones((4, 4), bool)
    intr = (32.0, 32.0, 1.5, 1.5)
    r, ref = run_both(n, mask, intr, theta_deg=5.0)
    assert r.partition0.component_count == 2
    assert r.partition0.labels[0] == 0
    assert_parity(r, ref, mask, intr)


def test_uniform_map_one_component():
    """test_graph.py:135-140: a uniform map is one component."""
    n = np.broadcast_to(_tilted(20.0, 30.0), (9, 13, 3)).copy()
    mask = np.ones((9, 13), bool)
    intr = (104.0, 104.0, 6.0, 4.0)
    r, ref = run_both(n, mask, intr)
    assert r.partition0.component_count == 1
    assert_parity(r, ref, mask, intr)


def test_theta_none_one_pixel_per_component():
    """graph.py:153-155 / test_graph.py:143-150: theta_c = None puts every
    valid pixel in its own component."""
    rng = np.random.default_rng(5)
    sc = scenes.voronoi_ortho("t", 6, 7, 3, 5, 0.2)
    mask = rng.random((6, 7)) < 0.8
    r, ref = run_both(sc.normals, mask, sc.intrinsics(), theta_deg=None)
    assert r.partition0.component_count == int(mask.sum())
    assert_parity(r, ref, mask, sc.intrinsics())


def test_fronto_parallel_plane_is_flat():
    """test_pipeline.py:14-23: a fronto-parallel plane integrates to a
    constant depth (every residual below 1e-8)."""
    n = np.broadcast_to(_tilted(0.0), (24, 40, 3)).copy()
    mask = np.ones((24, 40), bool)
    intr = (320.0, 320.0, 19.5, 11.5)
    r, ref = run_both(n, mask, intr)
    z = r.log_depth.values[mask]
    assert float(z.max() - z.min()) < 1e-8
    assert_parity(r, ref, mask, intr)


@pytest.mark.parametrize("shape", [(1, 7), (7, 1), (2, 2), (3, 31), (29, 61), (31, 33),
                                   (33, 97), (45, 130)])
def test_ragged_shapes(shape):
    """Maps narrower or shorter than one strip and widths that are not a
    multiple of the 30-column strip, with holes in the mask."""
    h, w = shape
    rng = np.random.default_rng(h * 1000 + w)
    cells = max(2, min(6, h * w // 40))
    sc = scenes.voronoi_ortho("ragged", h, w, cells, h + w, 0.2)
    mask = rng.random((h, w)) < 0.9
    if mask.sum() < 2:
        mask[:] = True
    r, ref = run_both(sc.normals, mask, sc.intrinsics())
    assert_parity(r, ref, mask, sc.intrinsics())


def test_single_valid_pixel():
    """One valid pixel: one singleton component, no edges, nothing to fill."""
    sc = scenes.voronoi_ortho("one", 5, 5, 2, 9, 0.2)
    mask = np.zeros((5, 5), bool)
    mask[2, 3] = True
    r, ref = run_both(sc.normals, mask, sc.intrinsics())
    assert r.partition0.component_count == 1
    assert_parity(r, ref, mask, sc.intrinsics())


def test_isolated_pixels_4conn():
    """A checkerboard mask at 4-connectivity has no edges: every pixel is a
    singleton component and the fill skips all of them (solver.py:220)."""
    sc = scenes.voronoi_ortho("checker", 20, 23, 3, 4, 0.2)
    v, u = np.mgrid[:20, :23]
    mask = (u + v) % 2 == 0
    r, ref = run_both(sc.normals, mask, sc.intrinsics(), connectivity=4)
    assert r.partition0.component_count == int(mask.sum())
    assert_parity(r, ref, mask, sc.intrinsics())


def test_bini_model_4conn_ragged():
    """The BiNI continuity model (4-connectivity only) on a ragged map."""
    sc = scenes.voronoi_ortho("bini", 37, 53, 5, 12, 0.2)
    r, ref = run_both(sc.normals, sc.mask, sc.intrinsics(), connectivity=4, model="bini")
    assert_parity(r, ref, sc.mask, sc.intrinsics())


def test_batch_bit_identical_to_single_maps():
    """Every reduction of a map (fill slots, unit sums, scale CG, energies,
    median) runs in an order that does not depend on the other maps of the
    batch, so a 12-map batch reproduces each map's single run bit for bit."""
    maps = [scenes.voronoi_ortho(f"s{i}", 70, 95, 5, 40 + i, 0.2) for i in range(12)]
    nms = [nb.NormalMap.create(m.normals, m.mask) for m in maps]
    intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
    theta = float(np.deg2rad(3.5))
    batch = nb.run_pipeline_batch(nb.stack(nms), intr, theta, nb.SolveSettings(freq_merging=3))
    for m, nm, i, b in zip(maps, nms, intr, batch):
        s = nb.run_pipeline(nm, i, theta, nb.SolveSettings(freq_merging=3))
        assert b.iterations == s.iterations
        assert np.array_equal(b.partition.labels, s.partition.labels)
        assert np.array_equal(b.filled.values, s.filled.values)
        assert np.array_equal(b.log_depth.values, s.log_depth.values)
        assert b.energies == s.energies


def test_stream_matches_batch():
    """run_pipeline_stream (overlapped upload / read-back) returns exactly
    run_pipeline_batch's results for every batch of the stream."""
    maps = [scenes.voronoi_ortho(f"st{i}", 48, 64, 4, 70 + i, 0.2) for i in range(3)]
    n = torch.from_numpy(np.stack([m.normals for m in maps])).pin_memory()
    mk = torch.from_numpy(np.stack([m.mask for m in maps])).pin_memory()
    intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
    theta = float(np.deg2rad(3.5))
    ref = nb.run_pipeline_batch(nb.NormalMap.create(n, mk), intr, theta)
    outs = list(nb.run_pipeline_stream(((n, mk) for _ in range(3)), intr, theta))
    assert len(outs) == 3
    for res, host in outs:
        assert host.is_pinned() and tuple(host.shape) == (3, 48 * 64)
        for i, (a, b) in enumerate(zip(ref, res)):
            assert a.iterations == b.iterations
            assert np.array_equal(a.log_depth.values, b.log_depth.values)
            assert np.array_equal(host[i].numpy(), a.log_depth.values_t.cpu().numpy())


def test_copy_to_host_kernel_ragged_and_errors():
    """ni_copy_to_host (the serving read-back through mapped pinned memory):
    exact bytes for lengths / offsets that exercise the unaligned head and the
    tail, nothing written past the range, and a loud error for pageable or
    misaligned destinations."""
    import ctypes as C

    from paper_2510_11508_b200 import _lib

    lib = _lib.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    src = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda")
    for off, n in ((0, 1 << 20), (3, 1000), (16, 17), (5, 7), (0, 0), (1, (1 << 20) - 1)):
        dst = torch.full((1 << 20,), 0xAB, dtype=torch.uint8).pin_memory()
        _lib.check(lib.ni_copy_to_host(C.c_void_p(src.data_ptr() + off),
                                       C.c_void_p(dst.data_ptr() + off), n, 7, s), "copy")
        torch.cuda.synchronize()
        want = torch.full((1 << 20,), 0xAB, dtype=torch.uint8)
        want[off:off + n] = src[off:off + n].cpu()
        assert torch.equal(dst, want), (off, n)
    pageable = torch.empty(1024, dtype=torch.uint8)
    assert lib.ni_copy_to_host(C.c_void_p(src.data_ptr()), C.c_void_p(pageable.data_ptr()),
                               1024, 4, s) != 0
    assert b"pinned" in lib.ni_last_error()
    dst = torch.empty(1024, dtype=torch.uint8).pin_memory()
    assert lib.ni_copy_to_host(C.c_void_p(src.data_ptr() + 1), C.c_void_p(dst.data_ptr()),
                               64, 4, s) != 0


def test_copy_from_host_kernel_and_stream_upload():
    """ni_copy_from_host (the upload twin of ni_copy_to_host): exact bytes for
    ragged ranges, a loud error for a pageable source, and a serving stream
    that uploads with it returns the copy-engine stream's results bit for bit."""
    import ctypes as C

    import paper_2510_11508_b200 as nb
    from paper_2510_11508_b200 import _lib, pipeline, scenes

    lib = _lib.load()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    src = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8).pin_memory()
    for off, n in ((0, 1 << 20), (3, 1000), (16, 17), (5, 7), (0, 0)):
        dst = torch.full((1 << 20,), 0xAB, dtype=torch.uint8, device="cuda")
        _lib.check(lib.ni_copy_from_host(C.c_void_p(dst.data_ptr() + off),
                                         C.c_void_p(src.data_ptr() + off), n, 5, s), "copy")
        torch.cuda.synchronize()
        want = torch.full((1 << 20,), 0xAB, dtype=torch.uint8)
        want[off:off + n] = src[off:off + n]
        assert torch.equal(dst.cpu(), want), (off, n)
    pageable = torch.empty(1024, dtype=torch.uint8)
    dst = torch.empty(1024, dtype=torch.uint8, device="cuda")
    assert lib.ni_copy_from_host(C.c_void_p(dst.data_ptr()), C.c_void_p(pageable.data_ptr()),
                                 1024, 4, s) != 0
    assert b"pinned" in lib.ni_last_error()

    maps = [scenes.config3(40 + i, size=48, cells=5) for i in range(3)]
    n = torch.from_numpy(np.stack([m.normals for m in maps]).astype(np.float32)).pin_memory()
    k = torch.from_numpy(np.stack([m.mask for m in maps])).pin_memory()
    intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
    theta = float(np.deg2rad(3.5))
    outs = {}
    for ctas in (0, 2):
        pipeline._H2D_CTAS = ctas
        try:
            outs[ctas] = [h.clone() for _, h in nb.run_pipeline_stream(((n, k) for _ in range(2)),
                                                                       intr, theta)]
        finally:
            pipeline._H2D_CTAS = 0
    for a, b in zip(outs[0], outs[2]):
        assert torch.equal(a, b)


def test_tail_kernel_matches_per_level_launches():
    """The single-launch tail of the multigrid fill (the small levels in one
    CTA) computes exactly what the per-level kernels compute: the same run
    with NI_MG_TAIL=0 (a process-wide knob, hence the subprocesses) gives a
    bit-identical log-depth."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import hashlib, numpy as np, paper_2510_11508_b200 as nb\n"
        "from paper_2510_11508_b200 import scenes\n"
        "sc = scenes.config4(3, size=160, cells=9)\n"
        "r = nb.run_pipeline(nb.NormalMap.create(sc.normals, sc.mask),\n"
        "                    nb.CameraIntrinsics(*sc.intrinsics()), float(np.deg2rad(3.5)),\n"
        "                    nb.SolveSettings(freq_merging=5))\n"
        "print('DIGEST', hashlib.sha256(r.log_depth.values.tobytes()).hexdigest(),\n"
        "      hashlib.sha256(r.filled.values.tobytes()).hexdigest(), r.iterations,\n"
        "      r.fill_report['mg']['levels'])\n")
    digests = []
    for tail in ("1", "0"):
        env = dict(os.environ, NI_MG_TAIL=tail)
        out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                             text=True, timeout=280)
        assert out.returncode == 0, out.stderr[-2000:]
        digests.append([ln for ln in out.stdout.splitlines() if ln.startswith("DIGEST")][0])
    assert digests[0] == digests[1], digests
    assert int(digests[0].split()[-1]) >= 3  # the case has levels for the tail to cover


def test_paired_weighted_fill_batch_vs_oracle():
    """A batch of >= 10 maps puts two components into one item of the weighted
    CG (ni_fill's paired mode, default mailbox depth): the refill pass of such
    a batch is compared with the oracle map by map (labels, outer iterations,
    merged partition, depth) -- not only with the unpaired GPU path."""
    maps = [scenes.config3(70 + i, size=56, cells=6) for i in range(12)]
    theta = float(np.deg2rad(3.5))
    st = nb.SolveSettings(freq_merging=5, refill_reweighted=True)
    nm = nb.NormalMap.create(np.stack([m.normals for m in maps]), np.stack([m.mask for m in maps]))
    res = nb.run_pipeline_batch(nm, [nb.CameraIntrinsics(*m.intrinsics()) for m in maps], theta, st)
    for m, r in zip(maps, res):
        ref = O.run_pipeline(m.normals.astype(np.float64), m.mask, m.intrinsics(), theta,
                             O.Settings(freq_merging=5, refill_reweighted=True))
        assert np.array_equal(r.partition0.labels, ref.labels0)
        assert r.iterations == ref.iterations
        assert np.array_equal(r.partition.labels, ref.labels)
        assert_depth_close(r.log_depth.values, ref.log_depth, m.mask, m.intrinsics()[0])


def test_theta_none_above_the_block_cg_limit():
    """theta_c = None on a map with more than 8192 valid pixels: every pixel is
    a component (graph.py:153-155), so the scale system has > 8192 unknowns
    and its CG takes the cooperative multi-block path; a few outer iterations
    against the oracle (labels, energies, depth)."""
    sc = scenes.config3(9, size=128, cells=8)
    assert int(sc.mask.sum()) > 8192
    st = nb.SolveSettings(max_iters=4)
    r = nb.run_pipeline(nb.NormalMap.create(sc.normals, sc.mask),
                        nb.CameraIntrinsics(*sc.intrinsics()), None, st)
    ref = O.run_pipeline(sc.normals.astype(np.float64), sc.mask, sc.intrinsics(), None,
                         O.Settings(max_iters=4))
    assert r.partition0.component_count == int(sc.mask.sum()) == ref.count0
    assert np.array_equal(r.partition0.labels, ref.labels0)
    assert r.iterations == ref.iterations
    np.testing.assert_allclose(r.energies, ref.energies, rtol=2e-3, atol=1e-9)
    assert len(r.warnings) == len(ref.warnings)
    assert_depth_close(r.log_depth.values, ref.log_depth, sc.mask, sc.intrinsics()[0])

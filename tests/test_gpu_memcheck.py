"""Memory discipline of the CUDA path without compute-sanitizer (closed on
the GPU pool): every device buffer the pipeline hands to a kernel is
poisoned (NaN / -1) and fenced by canary guard regions
(paper_2510_11508_b200/devmem.py).  A kernel reading a byte it did not write
changes the bit-exact result; one writing outside its buffer trips a
canary.  Covers the multigrid fill, the scale loop with merges, the
reweighted refill, the pixel baseline (the round-1 CG kernel's weighted
variant), BiNI at 4-connectivity, theta_c = None and a 12-map batch."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import devmem, scenes  # noqa: E402

THETA = float(np.deg2rad(3.5))


def _cases():
    c4 = scenes.config4(3, size=96, cells=14)
    c2 = scenes.config2(1, h=80, w=96, f=580.0, frac=0.4)
    batch = [scenes.voronoi_ortho(f"s{i}", 70, 95, 5, 40 + i, 0.2) for i in range(12)]
    return {
        "c4_merge_refill": lambda: [nb.run_pipeline(
            nb.NormalMap.create(c4.normals, c4.mask), nb.CameraIntrinsics(*c4.intrinsics()),
            THETA, nb.SolveSettings(freq_merging=5, refill_reweighted=True))],
        "c2_bini4": lambda: [nb.run_pipeline(
            nb.NormalMap.create(c2.normals, c2.mask), nb.CameraIntrinsics(*c2.intrinsics()),
            THETA, None, None, 4, "bini")],
        "theta_none": lambda: [nb.run_pipeline(
            nb.NormalMap.create(c4.normals[:24, :20], c4.mask[:24, :20]),
            nb.CameraIntrinsics(*c4.intrinsics()), None, nb.SolveSettings(max_iters=8))],
        "pixel_baseline": lambda: [nb.run_pixel_baseline(
            nb.NormalMap.create(c2.normals, c2.mask), nb.CameraIntrinsics(*c2.intrinsics()),
            nb.SolveSettings(max_iters=5))],
        "batch12": lambda: nb.run_pipeline_batch(
            nb.stack([nb.NormalMap.create(m.normals, m.mask) for m in batch]),
            [nb.CameraIntrinsics(*m.intrinsics()) for m in batch], THETA,
            nb.SolveSettings(freq_merging=3)),
    }


@pytest.mark.parametrize("name", sorted(_cases()))
def test_poisoned_and_guarded_run_is_bit_identical(name):
    run = _cases()[name]
    ref = run()
    with devmem.checking():
        got = run()
        nbuf = devmem.verify()
    assert nbuf > 0
    for a, b in zip(ref, got):
        assert a.iterations == b.iterations
        assert np.array_equal(a.log_depth.values, b.log_depth.values)
        if hasattr(a, "partition"):
            assert np.array_equal(a.partition.labels, b.partition.labels)
            assert np.array_equal(a.filled.values, b.filled.values)

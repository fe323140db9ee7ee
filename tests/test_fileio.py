"""File formats at the boundary vs files written by the reference
(tests/golden/files/, made by tests/golden/make_files_golden.py)."""

import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

FILES = os.path.join(GOLDEN, "files")


def expected():
    return dict(np.load(os.path.join(GOLDEN, "files_expected.npz")))


def test_pfm_round_trip_and_bytes(tmp_path):
    from paper_2510_11508_b200 import fileio

    arr = fileio.read_pfm(os.path.join(FILES, "normals.pfm"))
    assert arr.dtype == np.float32 and arr.shape == (37, 45, 3)
    out = tmp_path / "n.pfm"
    fileio.write_pfm(out, arr)
    assert out.read_bytes() == open(os.path.join(FILES, "normals.pfm"), "rb").read()
    depth, mask = fileio.read_depth(os.path.join(FILES, "depth_gt.pfm"))
    assert np.array_equal(depth, expected()["depth"])
    out2 = tmp_path / "d.pfm"
    fileio.write_depth(out2, depth, mask)
    assert out2.read_bytes() == open(os.path.join(FILES, "depth_gt.pfm"), "rb").read()


def test_pfm_errors(tmp_path):
    from paper_2510_11508_b200 import errors, fileio

    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"P7\n3 3\n-1.0\n")
    with pytest.raises(errors.MalformedHeader):
        fileio.read_pfm(bad)
    short = tmp_path / "short.pfm"
    short.write_bytes(b"Pf\n3 3\n-1.0\n" + b"\x00" * 8)
    with pytest.raises(errors.TruncatedPayload):
        fileio.read_pfm(short)


def test_labels_blob_and_png_colors():
    from paper_2510_11508_b200 import fileio

    e = expected()
    lab, count, w, h = fileio.read_labels_bin(os.path.join(FILES, "labels.bin"))
    assert (w, h, count) == (45, 37, int(e["count"]))
    assert np.array_equal(lab, e["labels"])
    assert fileio.export_labels(lab, w, h) == open(os.path.join(FILES, "labels.bin"), "rb").read()
    assert np.array_equal(fileio.hash_colors(lab.reshape(h, w)), e["hash_rgb"])


def test_intrinsics_json(tmp_path):
    from paper_2510_11508_b200 import errors, fileio

    intr = fileio.load_intrinsics(os.path.join(FILES, "intrinsics.json"))
    out = tmp_path / "i.json"
    fileio.save_intrinsics(out, intr)
    assert out.read_text() == open(os.path.join(FILES, "intrinsics.json")).read()
    (tmp_path / "bad.json").write_text('{"fx": 1}')
    with pytest.raises(errors.MalformedHeader):
        fileio.load_intrinsics(tmp_path / "bad.json")


@pytest.mark.gpu
def test_png16_and_pfm_normals_decode_bit_exact():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2510_11508_b200 import fileio

    e = expected()
    nm = fileio.read_png16_normals(os.path.join(FILES, "normals.png"))
    assert np.array_equal(nm.mask, e["png_mask"])
    assert np.array_equal(nm.normals, e["png_normals"])
    nf = fileio.read_png16_normals(os.path.join(FILES, "normals.png"), flip_z=True)
    assert np.array_equal(nf.normals, e["png_flip_normals"])
    pf = fileio.read_normals_pfm(os.path.join(FILES, "normals.pfm"))
    assert np.array_equal(pf.normals, e["pfm_normals"]) and np.array_equal(pf.mask, e["pfm_mask"])
    nm2, intr, gt = fileio.load_scene_dir(FILES)
    assert np.array_equal(nm2.normals, e["scene_normals"])
    assert np.array_equal(nm2.mask, e["scene_mask"])
    assert [intr.fx, intr.fy, intr.cx, intr.cy] == list(e["scene_intr"])
    assert np.array_equal(gt, e["depth"])


@pytest.mark.gpu
def test_device_side_writers_match_the_host_formulas(tmp_path):
    """The writers that do their per-pixel arithmetic on the GPU produce the
    bytes the reference's host formulas produce: the normals PFM (rewriting
    the reference's own file byte for byte), the PNG16 quantisation, the
    depth PFM of a LogDepthMap, the label blob of a device Partition, and the
    pinned-memory stream writer."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2510_11508_b200 as nb
    from paper_2510_11508_b200 import fileio

    pf = fileio.read_normals_pfm(os.path.join(FILES, "normals.pfm"))
    fileio.write_normals_pfm(tmp_path / "n.pfm", pf)
    assert (tmp_path / "n.pfm").read_bytes() == open(os.path.join(FILES, "normals.pfm"),
                                                      "rb").read()
    nm = fileio.read_png16_normals(os.path.join(FILES, "normals.png"))
    fileio.write_png16_normals(tmp_path / "n.png", nm)
    import cv2
    got = cv2.imread(str(tmp_path / "n.png"), cv2.IMREAD_UNCHANGED)[..., ::-1]
    want = np.rint(np.clip((nm.normals + 1.0) * 0.5, 0.0, 1.0) * 65535.0).astype(np.uint16)
    want[~nm.mask] = 0
    assert np.array_equal(got, want)
    intr = fileio.load_intrinsics(os.path.join(FILES, "intrinsics.json"))
    res = nb.run_pipeline(pf, intr, float(np.deg2rad(3.5)))
    fileio.write_depth(tmp_path / "a.pfm", res.log_depth)
    fileio.write_depth(tmp_path / "b.pfm", nb.depth_from_logdepth(res.log_depth), pf.mask)
    assert (tmp_path / "a.pfm").read_bytes() == (tmp_path / "b.pfm").read_bytes()
    h, w = pf.mask.shape
    assert fileio.export_labels(res.partition0, w, h) == \
        fileio.export_labels(res.partition0.labels, w, h)
    host = torch.from_numpy(np.stack([res.log_depth.values.reshape(-1)] * 2)).pin_memory()
    with fileio.DepthStreamWriter(h, w) as wr:
        wr.submit([tmp_path / "s0.pfm", tmp_path / "s1.pfm"], host, np.stack([pf.mask] * 2))
    fileio.write_depth(tmp_path / "c.pfm", np.exp(res.log_depth.values), pf.mask)
    for p in ("s0.pfm", "s1.pfm"):
        assert (tmp_path / p).read_bytes() == (tmp_path / "c.pfm").read_bytes()

"""File-format fixtures written and read back by the REAL reference
(fileio.py, graph.py:253-275), in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_files_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "files")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2510_11508_b200 import scenes  # noqa: E402

import normint  # noqa: E402
from normint import fileio as F  # noqa: E402
from normint import graph as G  # noqa: E402
from normint.geometry import CameraIntrinsics, NormalMap  # noqa: E402


def main():
    os.makedirs(OUT, exist_ok=True)
    sc = scenes.config2(21, h=37, w=45, f=300.0, frac=0.5)
    nm = NormalMap.create(sc.normals.astype(np.float64), sc.mask)
    noisy = normint.perturb_normals(nm, np.deg2rad(3.0), 4)
    F.write_normals_pfm(os.path.join(OUT, "normals.pfm"), nm)
    F.write_png16_normals(os.path.join(OUT, "normals.png"), noisy)
    F.write_mask(os.path.join(OUT, "mask.png"), sc.mask)
    depth = np.where(sc.mask, 1000.0 + np.arange(sc.mask.size).reshape(sc.mask.shape) * 0.37, 0.0)
    F.write_depth(os.path.join(OUT, "depth_gt.pfm"), depth, sc.mask)
    F.save_intrinsics(os.path.join(OUT, "intrinsics.json"), CameraIntrinsics(*sc.intrinsics()))
    g = G.build_pixel_graph(nm, 8)
    p = G.form_components(g, nm, float(np.deg2rad(3.5)))
    F.write_labels_bin(os.path.join(OUT, "labels.bin"), p, 45, 37)
    F.write_labels_png(os.path.join(OUT, "labels.png"), p, 45, 37)
    png = F.read_png16_normals(os.path.join(OUT, "normals.png"))
    png_flip = F.read_png16_normals(os.path.join(OUT, "normals.png"), flip_z=True)
    pfm = F.read_normals_pfm(os.path.join(OUT, "normals.pfm"))
    scene = F.load_scene_dir(OUT)
    np.savez_compressed(
        os.path.join(HERE, "files_expected.npz"),
        png_normals=png.normals, png_mask=png.mask, png_flip_normals=png_flip.normals,
        pfm_normals=pfm.normals, pfm_mask=pfm.mask, labels=p.labels.astype(np.int64),
        count=p.component_count, depth=F.read_depth(os.path.join(OUT, "depth_gt.pfm"))[0],
        scene_normals=scene[0].normals, scene_mask=scene[0].mask,
        scene_intr=np.array([scene[1].fx, scene[1].fy, scene[1].cx, scene[1].cy]),
        hash_rgb=F._hash_colors(p.labels.reshape(37, 45)))
    print("written", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_2510_11508_b200 as nb
from paper_2510_11508_b200 import scenes
sc = scenes.config3(2, size=64, cells=6)
nm = nb.NormalMap.create(sc.normals, sc.mask)
try:
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), float(np.deg2rad(3.5)))
    print("ok", r.iterations)
except Exception as e:
    print("ERR", e)

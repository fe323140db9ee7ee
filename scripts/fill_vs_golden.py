"""One config through run_pipeline against its full-size reference fixture: outer
iterations, energies, and how far the filled state / depth samples are from the
reference's (used to compare multigrid cycle variants, NI_MG_W_LO / NI_MG_W_HI).

    python scripts/fill_vs_golden.py C4
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
d = dict(np.load(os.path.join("tests", "golden", "full", name + ".npz"), allow_pickle=False))
sc = scenes.config5_map(int(name[3:])) if name.startswith("C5_") else scenes.CONFIGS[name]()
st = nb.SolveSettings(freq_merging=sc.options.get("merge_freq"))
r = nb.run_pipeline(nb.NormalMap.create(sc.normals, sc.mask), nb.CameraIntrinsics(*sc.intrinsics()),
                    float(np.deg2rad(3.5)), st)
torch.cuda.synchronize()
idx = d["sample_idx"]
f = r.filled.values.reshape(-1)[idx]
z = r.log_depth.values.reshape(-1)[idx]
print(name, "W levels", os.environ.get("NI_MG_W_LO", "2"), "..", os.environ.get("NI_MG_W_HI", "3"),
      "iterations", r.iterations, "ref", int(d["iterations"]), "fill report", r.fill_report.get("mg"))
print(" filled: max |d|", float(np.abs(f - d["filled_s"]).max()), "rms",
      float(np.sqrt(np.mean((f - d["filled_s"]) ** 2))))
print(" depth : max |d|", float(np.abs(z - d["log_depth_s"]).max()))
e, er = np.array(r.energies), d["energies"]
k = min(len(e), len(er))
print(" energies rel diff:", np.array2string(np.abs(e[:k] - er[:k]) / np.maximum(np.abs(er[:k]), 1e-300),
                                             precision=2, max_line_width=200))
print(" fill iterations max", int(np.max(r.fill_iterations)))

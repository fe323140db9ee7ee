import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb
from paper_2510_11508_b200 import scenes
from oracle import normint_oracle as O
maps = [scenes.voronoi_ortho(f"s{i}", 70, 95, 5, 40 + i, 0.2) for i in range(12)]
nms = [nb.NormalMap.create(m.normals, m.mask) for m in maps]
intr = [nb.CameraIntrinsics(*m.intrinsics()) for m in maps]
theta = float(np.deg2rad(3.5))
st = nb.SolveSettings(freq_merging=3)
batch = nb.run_pipeline_batch(nb.stack(nms), intr, theta, st)
for k, (m, nm, i, b) in enumerate(zip(maps, nms, intr, batch)):
    s = nb.run_pipeline(nm, i, theta, st)
    o = O.run_pipeline(m.normals.astype(np.float64), m.mask, m.intrinsics(), theta, O.Settings(freq_merging=3))
    print(k, "comps", b.partition0.component_count, "iters batch/single/oracle", b.iterations, s.iterations, o.iterations)
    print("   E batch ", np.array(b.energies))
    print("   E single", np.array(s.energies))
    print("   E oracle", np.array(o.energies))

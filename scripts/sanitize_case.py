"""Small workloads for compute-sanitizer (scripts/sanitize.sh): a 96x96 C4
map with merges, a 12-map batch, the pixel baseline and the refill pass."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2510_11508_b200 as nb  # noqa: E402
from paper_2510_11508_b200 import scenes  # noqa: E402

theta = float(np.deg2rad(3.5))
sc = scenes.config4(3, size=96, cells=14)
nm = nb.NormalMap.create(sc.normals, sc.mask)
r = nb.run_pipeline(nm, nb.CameraIntrinsics(*sc.intrinsics()), theta,
                    nb.SolveSettings(freq_merging=5, refill_reweighted=True))
print("c4_96", r.iterations, r.partition.component_count)
maps = [scenes.voronoi_ortho(f"s{i}", 70, 95, 5, 40 + i, 0.2) for i in range(12)]
b = nb.run_pipeline_batch(nb.stack([nb.NormalMap.create(m.normals, m.mask) for m in maps]),
                          [nb.CameraIntrinsics(*m.intrinsics()) for m in maps], theta)
print("batch12", [x.iterations for x in b])
pb = nb.run_pixel_baseline(nm, nb.CameraIntrinsics(*sc.intrinsics()),
                           nb.SolveSettings(max_iters=4))
print("pixel baseline", pb.iterations)

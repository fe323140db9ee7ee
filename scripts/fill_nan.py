import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_2510_11508_b200 as nb
from paper_2510_11508_b200 import _lib
d = dict(np.load('tests/golden/sine_ref.npz'))
nm = nb.NormalMap.create(d['normals'], d['mask'])
for rep in range(3):
    r = nb.run_pipeline(nm, nb.CameraIntrinsics(*d['intr']), float(np.deg2rad(3.5)))
    f = r.filled.values
    lab = r.partition0.labels.reshape(f.shape)
    bad = ~np.isfinite(f)
    print('rep', rep, 'nan px', bad.sum(), 'comps', np.unique(lab[bad])[:10], _lib.fill_report())
    err = np.abs(f - d['filled'])[d['mask']]
    print('  max err finite', np.nanmax(err), 'iters max', r.fill_iterations.max())
    if bad.any():
        ys, xs = np.nonzero(bad); print('  rows', ys.min(), ys.max(), 'cols', xs.min(), xs.max())

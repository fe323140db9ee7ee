"""Generate the golden fixtures by running the REAL reference ``normint``.

Run in the build container only (the reference does not exist on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each case is a small seeded scene from ``paper_2510_11508_b200.scenes`` (the
BASELINE config generators at reduced size) or one of the reference's own
analytic scenes.  The float32 normals handed to the GPU are stored; the
reference sees ``NormalMap.create(n32.astype(float64), mask)`` exactly as its
PFM reader would build it (fileio.py:118-123).  Outputs: ``normint.run_pipeline``
results plus, for the ``seam_*`` cases, the per-seam outputs of
``form_components`` / ``build_edge_coefficients`` / ``fill_components`` /
``relative_scale_step`` / ``merge_components``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2510_11508_b200 import scenes  # noqa: E402

import normint  # noqa: E402
from normint import graph as ngraph  # noqa: E402
from normint import continuity as ncont  # noqa: E402
from normint import solver as nsolver  # noqa: E402
from normint.geometry import CameraIntrinsics, NormalMap  # noqa: E402
from normint.synth import SceneSpec, render_scene  # noqa: E402


def _scene_case(sc):
    return sc.normals, sc.mask, (sc.fx, sc.fy, sc.cx, sc.cy)


def _ref_scene(kind, size, noise=0.0, seed=0):
    r = render_scene(SceneSpec(kind, size, size))
    nm = r.normal_map
    if noise:
        nm = normint.perturb_normals(nm, np.deg2rad(noise), seed)
    n32 = nm.normals.astype(np.float32)
    n32[~nm.mask] = 0
    i = r.intrinsics
    return n32, nm.mask.copy(), (i.fx, i.fy, i.cx, i.cy)


CASES = {
    # name: (scene factory, options)
    "c1_hemi64": (lambda: _scene_case(scenes.config1(0, size=64, radius=20.0, step=5.0)), {}),
    "c2_blob_96x80": (lambda: _scene_case(scenes.config2(1, h=80, w=96, f=580.0, frac=0.4)), {}),
    "c3_voronoi64": (lambda: _scene_case(scenes.config3(2, size=64, cells=6)), {}),
    "c4_voronoi96_merge": (lambda: _scene_case(scenes.config4(3, size=96, cells=14)), {"merge_freq": 5}),
    "c5_voronoi48": (lambda: _scene_case(scenes.config5_map(0, size=48, cells=5)), {}),
    "c3_voronoi64_conn4": (lambda: _scene_case(scenes.config3(2, size=64, cells=6)), {"connectivity": 4}),
    "bini_conn4": (lambda: _scene_case(scenes.config2(5, h=64, w=72, f=450.0, frac=0.5)),
                   {"connectivity": 4, "model": "bini"}),
    "hard_mode": (lambda: _scene_case(scenes.config3(7, size=56, cells=5, sigma_deg=0.5)), {"reweighting": "hard"}),
    "off_mode_merge2": (lambda: _scene_case(scenes.config3(8, size=56, cells=7, sigma_deg=0.5)),
                        {"reweighting": "off", "merge_freq": 2}),
    "bump_ref_merge": (lambda: _ref_scene("sphere_on_plane", 64, 0.2, 3), {"merge_freq": 5}),
    "sine_ref": (lambda: _ref_scene("sine_relief", 48), {}),
    "theta_none_16": (lambda: _ref_scene("sphere_patch", 16), {"theta_c_deg": None}),
    "gauge_depth": (lambda: _scene_case(scenes.config1(4, size=40, radius=12.0, step=3.0, sigma_deg=0.3)),
                    {"gauge_depth": 2.5}),
    "theta2_noisy": (lambda: _scene_case(scenes.config2(9, h=60, w=64, f=420.0, frac=0.6)), {"theta_c_deg": 2.0}),
    # second fill pass with bilateral weights at the filled state (solver.py:237-238)
    "refill_voronoi48": (lambda: _scene_case(scenes.config5_map(3, size=48, cells=5)), {"refill": True}),
    "refill_bump_merge": (lambda: _ref_scene("sphere_on_plane", 48, 0.2, 5), {"refill": True, "merge_freq": 5}),
}

# run_pixel_baseline (pipeline.py:297-369) cases
BASELINE_CASES = {
    "pb_hemi40": (lambda: _scene_case(scenes.config1(0, size=40, radius=12.0, step=3.0)), {}),
    "pb_voronoi40": (lambda: _scene_case(scenes.config3(2, size=40, cells=4)), {}),
    "pb_blob_conn4_bini": (lambda: _scene_case(scenes.config2(5, h=40, w=48, f=300.0, frac=0.5)),
                           {"connectivity": 4, "model": "bini"}),
    "pb_hard_gauge": (lambda: _scene_case(scenes.config3(7, size=36, cells=4, sigma_deg=0.5)),
                      {"reweighting": "hard", "gauge_depth": 3.0}),
    "pb_patch_ref": (lambda: _ref_scene("sphere_patch", 32), {}),
}


def run_case(name, factory, opts):
    n32, mask, intr = factory()
    theta = opts.get("theta_c_deg", 3.5)
    conn = opts.get("connectivity", 8)
    model = opts.get("model", "milano")
    settings = nsolver.SolveSettings(freq_merging=opts.get("merge_freq"), worker_count=1,
                                     refill_reweighted=bool(opts.get("refill", False)))
    weights = ncont.WeightParams(reweighting_mode=opts.get("reweighting", "soft"))
    nm = NormalMap.create(n32.astype(np.float64), mask)
    cam = CameraIntrinsics(*intr)
    res = normint.run_pipeline(nm, cam, None if theta is None else float(np.deg2rad(theta)),
                               settings, weights, conn, model, opts.get("gauge_depth"))
    rec = [{k: v for k, v in r.items() if k != "wall_ms"} for r in res.records]
    out = dict(
        normals=n32, mask=mask, intr=np.array(intr, np.float64),
        labels0=res.partition0.labels.astype(np.int32), count0=res.partition0.component_count,
        labels=res.partition.labels.astype(np.int32), count=res.partition.component_count,
        filled=res.filled.values, log_depth=res.log_depth.values,
        energies=np.array(res.energies), iterations=res.iterations,
        warnings=len(res.warnings), warning_text=json.dumps(res.warnings),
        options=json.dumps(opts), records=json.dumps(rec),
    )
    return out


def run_baseline_case(name, factory, opts):
    n32, mask, intr = factory()
    conn = opts.get("connectivity", 8)
    model = opts.get("model", "milano")
    settings = nsolver.SolveSettings(worker_count=1)
    weights = ncont.WeightParams(reweighting_mode=opts.get("reweighting", "soft"))
    nm = NormalMap.create(n32.astype(np.float64), mask)
    cam = CameraIntrinsics(*intr)
    res = normint.run_pixel_baseline(nm, cam, settings, weights, conn, model, opts.get("gauge_depth"))
    rec = [{k: v for k, v in r.items() if k != "wall_ms"} for r in res.records]
    return dict(
        normals=n32, mask=mask, intr=np.array(intr, np.float64), log_depth=res.log_depth.values,
        energies=np.array(res.energies), iterations=res.iterations, warnings=len(res.warnings),
        warning_text=json.dumps(res.warnings), options=json.dumps(opts), records=json.dumps(rec),
    )


def seam_case():
    """Per-seam outputs on one small noisy scene (32x32 Voronoi, 8-conn)."""
    n32, mask, intr = _scene_case(scenes.config3(11, size=32, cells=4, sigma_deg=0.5))
    nm = NormalMap.create(n32.astype(np.float64), mask)
    cam = CameraIntrinsics(*intr)
    g = ngraph.build_pixel_graph(nm, 8)
    p = ngraph.form_components(g, nm, float(np.deg2rad(3.5)))
    co = ncont.build_edge_coefficients(nm, g, cam, "milano")
    st = nsolver.SolveSettings(worker_count=1)
    wp = ncont.WeightParams()
    z, _ = nsolver.fill_components(p, g, co, wp, st)
    q = ngraph.build_quotient(g, p)
    zc = z.copy()
    steps = {}
    for t in (0, 2):
        s = nsolver.relative_scale_step(q, p, zc, t, st, wp, co)
        steps[t] = s
        if p.component_count:
            zc[p.labels >= 0] += s.scales[p.labels[p.labels >= 0]]
    merged = ngraph.merge_components(q, p, np.abs(steps[2].residual[0::2]))
    return dict(
        normals=n32, mask=mask, intr=np.array(intr, np.float64),
        edges=g.edges.astype(np.int32), labels0=p.labels.astype(np.int32), count0=p.component_count,
        omega_a=co.omega_to_a, omega_b=co.omega_to_b, gamma_a=co.gamma_a, gamma_b=co.gamma_b,
        opp_a=co.opp_a.astype(np.int32), opp_b=co.opp_b.astype(np.int32), valid=co.valid,
        filled=z, inter_edge_ids=q.edge_ids.astype(np.int32),
        scales_t0=steps[0].scales, energy_t0=steps[0].energy, weights_t0=steps[0].weights,
        scales_t2=steps[2].scales, energy_t2=steps[2].energy, weights_t2=steps[2].weights,
        residual_t2=steps[2].residual,
        merged_labels=merged.labels.astype(np.int32), merged_count=merged.component_count,
    )


def main():
    out_dir = HERE
    only = set(sys.argv[1:])
    for name, (factory, opts) in BASELINE_CASES.items():
        if only and name not in only:
            continue
        d = run_baseline_case(name, factory, opts)
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), **d)
        print(f"{name}: {d['mask'].shape} valid={int(d['mask'].sum())} iters={d['iterations']}")
    for name, (factory, opts) in CASES.items():
        if only and name not in only:
            continue
        d = run_case(name, factory, opts)
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), **d)
        print(f"{name}: {d['mask'].shape} valid={int(d['mask'].sum())} comps={d['count0']}->{d['count']} "
              f"iters={d['iterations']}")
    if only and "seam_voronoi32" not in only:
        return
    d = seam_case()
    np.savez_compressed(os.path.join(out_dir, "seam_voronoi32.npz"), **d)
    print("seam_voronoi32: comps", d["count0"], "edges", len(d["edges"]))


if __name__ == "__main__":
    main()

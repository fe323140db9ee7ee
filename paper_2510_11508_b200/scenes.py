"""Seeded synthetic normal maps for the five BASELINE.json configurations.

This is harness code (input generation), not part of the timed path.  The
reference ships no generator for these shapes (its ``synth.py`` only renders
six analytic toy scenes, /root/reference/pkg/src/normint/synth.py:1-25), so
the generators below follow SURVEY.md §8(d):

* C1  256x256 orthographic hemisphere (r=80 px) raised +20 px on a plane, full
      mask, no noise, seed 0.
* C2  612x512 perspective (f=3700), ~15 % smooth blob mask, depth 1500 + 8
      Gaussian bumps + 2 occluding steps, 0.5 deg noise, seed 1.
* C3  2048x2048 orthographic, disk mask (~3.0 M px), 32 Voronoi cells of tilted
      paraboloids offset by depth steps, 0.2 deg noise, seed 2.
* C4  4096x4096 perspective (f=4000), ellipse mask (~12 M px), 128 Voronoi
      cells, 0.5 deg noise, seed 3; run with merging every 5 iterations.
* C5  64 maps of 1024x1024 orthographic, seeds 100..163, 16 Voronoi cells,
      full mask, 0.2 deg noise.

Orthographic configs use the pinhole stand-in of SURVEY.md (D1): the reference
is pinhole-only, so the camera is f = D = 8*max(W, H) px with the
principal point at the image centre and depth z = D - h, h being the height
towards the camera in pixel units.  Normals are evaluated analytically from
the perspective surface p(u, v) = z(u, v) * tau(u, v) in float64 and stored as
float32; the same float32 bits go to the CPU oracle and to the GPU.

Every array is produced from ``numpy.random.default_rng(seed)`` (PCG64) so the
inputs are identical on every machine.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Scene:
    """A generated normal map plus the options the config is run with."""

    name: str
    normals: np.ndarray  # (H, W, 3) float32, zero on invalid pixels
    mask: np.ndarray  # (H, W) bool
    fx: float
    fy: float
    cx: float
    cy: float
    depth: np.ndarray  # (H, W) float64 ground-truth depth (0 outside mask)
    options: dict = field(default_factory=dict)

    @property
    def height(self) -> int:
        return self.mask.shape[0]

    @property
    def width(self) -> int:
        return self.mask.shape[1]

    @property
    def valid_count(self) -> int:
        return int(self.mask.sum())

    def intrinsics(self):
        return (self.fx, self.fy, self.cx, self.cy)


# --------------------------------------------------------------------------
# geometry helpers


def _normals_from_depth(z, z_u, z_v, fx, fy, cx, cy):
    """Unit normals of p = z * tau with tau = ((u-cx)/fx, (v-cy)/fy, 1).

    p_u = z_u tau + z (1/fx, 0, 0) and p_v = z_v tau + z (0, 1/fy, 0); the
    normal is their cross product oriented to face the camera (n . tau < 0).
    """
    h, w = z.shape
    v, u = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64), indexing="ij")
    a = (u - cx) / fx
    b = (v - cy) / fy
    pu = np.stack([z_u * a + z / fx, z_u * b, z_u], axis=-1)
    pv = np.stack([z_v * a, z_v * b + z / fy, z_v], axis=-1)
    n = np.cross(pu, pv)
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    facing = n[..., 0] * a + n[..., 1] * b + n[..., 2]
    n[facing > 0] *= -1.0
    return n


def _tilt_normals(n, mask, sigma_deg, rng):
    """Rotate every valid normal by |N(0, sigma)| about a random tangent axis.

    Same noise model as the reference's ``perturb_normals``
    (synth.py:296-325): the tilt angle is half-normal, the tangent direction
    uniform.  Implemented with Rodrigues' formula on the tangent axis.
    """
    if sigma_deg <= 0:
        return n
    sig = np.deg2rad(sigma_deg)
    m = n[mask]
    cnt = len(m)
    ang = np.abs(rng.normal(0.0, sig, size=cnt))
    phi = rng.uniform(0.0, 2.0 * np.pi, size=cnt)
    ref = np.zeros_like(m)
    use_x = np.abs(m[:, 0]) < 0.9
    ref[use_x, 0] = 1.0
    ref[~use_x, 1] = 1.0
    t1 = np.cross(m, ref)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(m, t1)
    axis = np.cos(phi)[:, None] * t1 + np.sin(phi)[:, None] * t2
    rot = np.cos(ang)[:, None] * m + np.sin(ang)[:, None] * np.cross(axis, m)
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    out = n.copy()
    out[mask] = rot
    return out


def _finish(name, z, z_u, z_v, mask, fx, fy, cx, cy, sigma_deg, rng, options):
    n = _normals_from_depth(z, z_u, z_v, fx, fy, cx, cy)
    n = _tilt_normals(n, mask, sigma_deg, rng)
    n[~mask] = 0.0
    n32 = n.astype(np.float32)
    depth = np.where(mask, z, 0.0)
    return Scene(name, n32, mask.copy(), float(fx), float(fy), float(cx), float(cy), depth, options)


def _grid(h, w):
    return np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64), indexing="ij")


def _voronoi_height(h, w, cells, rng):
    """Voronoi partition into tilted paraboloid patches offset by steps.

    Each cell: h = off + g . d + kappa |d|^2, d = (u, v) - site,
    kappa ~ U[-1e-3, 1e-3], |g| = tan(theta), theta ~ U[0, 40 deg],
    off ~ U[5, 50] so every cell boundary is a depth step.
    """
    sites = np.stack([rng.uniform(0, w, cells), rng.uniform(0, h, cells)], axis=1)
    off = rng.uniform(5.0, 50.0, cells)
    theta = np.deg2rad(rng.uniform(0.0, 40.0, cells))
    phi = rng.uniform(0.0, 2.0 * np.pi, cells)
    gx = np.tan(theta) * np.cos(phi)
    gy = np.tan(theta) * np.sin(phi)
    kap = rng.uniform(-1e-3, 1e-3, cells)
    hh = np.empty((h, w))
    hu = np.empty((h, w))
    hv = np.empty((h, w))
    u = np.arange(w, dtype=np.float64)
    rows = max(1, (1 << 22) // max(1, w * cells))
    for r0 in range(0, h, rows):
        r1 = min(h, r0 + rows)
        v = np.arange(r0, r1, dtype=np.float64)
        du = u[None, :, None] - sites[None, None, :, 0]
        dv = v[:, None, None] - sites[None, None, :, 1]
        cell = np.argmin(du * du + dv * dv, axis=2)
        duc = u[None, :] - sites[cell, 0]
        dvc = v[:, None] - sites[cell, 1]
        k = kap[cell]
        hh[r0:r1] = off[cell] + gx[cell] * duc + gy[cell] * dvc + k * (duc * duc + dvc * dvc)
        hu[r0:r1] = gx[cell] + 2.0 * k * duc
        hv[r0:r1] = gy[cell] + 2.0 * k * dvc
    return hh, hu, hv


# --------------------------------------------------------------------------
# configs


def config1(seed: int = 0, size: int = 256, radius: float = 80.0, step: float = 20.0,
            sigma_deg: float = 0.0) -> Scene:
    """256x256 orthographic hemisphere r=80 on a plane, +20 px rim step."""
    h = w = size
    rng = np.random.default_rng(seed)
    d = 8.0 * max(w, h)
    cx, cy = (w - 1) / 2, (h - 1) / 2
    v, u = _grid(h, w)
    rad = radius
    rho2 = (u - cx) ** 2 + (v - cy) ** 2
    inside = rho2 < rad * rad
    s = np.sqrt(np.where(inside, rad * rad - rho2, 1.0))
    hh = np.where(inside, step + s, 0.0)
    hu = np.where(inside, -(u - cx) / s, 0.0)
    hv = np.where(inside, -(v - cy) / s, 0.0)
    mask = np.ones((h, w), dtype=bool)
    return _finish("C1", d - hh, -hu, -hv, mask, d, d, cx, cy, sigma_deg, rng,
                   {"theta_c_deg": 3.5, "merge_freq": None})


def _blob_mask(h, w, frac, rng):
    v, u = _grid(h, w)
    f = np.zeros((h, w))
    for _ in range(6):
        cu, cv = rng.uniform(0.25 * w, 0.75 * w), rng.uniform(0.25 * h, 0.75 * h)
        s = rng.uniform(0.08, 0.16) * min(h, w)
        f += np.exp(-((u - cu) ** 2 + (v - cv) ** 2) / (2 * s * s))
    thr = np.quantile(f, 1.0 - frac)
    return f > thr


def config2(seed: int = 1, h: int = 512, w: int = 612, f: float = 3700.0,
            frac: float = 0.15) -> Scene:
    """612x512 perspective (f=3700) blob with Gaussian bumps and two steps."""
    rng = np.random.default_rng(seed)
    sc = w / 612.0
    cx, cy = (w - 1) / 2, (h - 1) / 2
    mask = _blob_mask(h, w, frac, rng)
    v, u = _grid(h, w)
    z = np.full((h, w), 1500.0)
    zu = np.zeros((h, w))
    zv = np.zeros((h, w))
    for _ in range(8):
        a = rng.uniform(20.0, 80.0) * sc
        s = rng.uniform(15.0, 60.0) * sc
        bu, bv = rng.uniform(0, w), rng.uniform(0, h)
        g = a * np.exp(-((u - bu) ** 2 + (v - bv) ** 2) / (2 * s * s))
        z += g
        zu += -g * (u - bu) / (s * s)
        zv += -g * (v - bv) / (s * s)
    for _ in range(2):
        step = rng.uniform(30.0, 100.0) * sc
        pu, pv = rng.uniform(0.3 * w, 0.7 * w), rng.uniform(0.3 * h, 0.7 * h)
        ang = rng.uniform(0.0, np.pi)
        side = (u - pu) * np.cos(ang) + (v - pv) * np.sin(ang) > 0
        z += np.where(side, step, 0.0)
    return _finish("C2", z, zu, zv, mask, f, f, cx, cy, 0.5, rng,
                   {"theta_c_deg": 3.5, "merge_freq": None})


def voronoi_ortho(name, h, w, cells, seed, sigma_deg, mask=None, merge_freq=None) -> Scene:
    rng = np.random.default_rng(seed)
    d = 8.0 * max(w, h)
    cx, cy = (w - 1) / 2, (h - 1) / 2
    hh, hu, hv = _voronoi_height(h, w, cells, rng)
    if mask is None:
        mask = np.ones((h, w), dtype=bool)
    return _finish(name, d - hh, -hu, -hv, mask, d, d, cx, cy, sigma_deg, rng,
                   {"theta_c_deg": 3.5, "merge_freq": merge_freq})


def config3(seed: int = 2, size: int = 2048, cells: int = 32, sigma_deg: float = 0.2) -> Scene:
    """2048^2 orthographic disk (~3.0 M px), 32 Voronoi paraboloid cells."""
    h = w = size
    v, u = _grid(h, w)
    r = 977.0 * size / 2048
    mask = (u - (w - 1) / 2) ** 2 + (v - (h - 1) / 2) ** 2 < r * r
    return voronoi_ortho("C3", h, w, cells, seed, sigma_deg, mask)


def config4(seed: int = 3, size: int = 4096, cells: int = 128, sigma_deg: float = 0.5) -> Scene:
    """4096^2 perspective (f=4000) ellipse (~12 M px), 128 Voronoi cells."""
    h = w = size
    sc = size / 4096
    rng = np.random.default_rng(seed)
    f = 4000.0 * sc
    cx, cy = (w - 1) / 2, (h - 1) / 2
    v, u = _grid(h, w)
    ea, eb = 2040.0 * sc, 1872.0 * sc
    mask = ((u - cx) / ea) ** 2 + ((v - cy) / eb) ** 2 < 1.0
    hh, hu, hv = _voronoi_height(h, w, cells, rng)
    z0 = f  # one depth unit per pixel at the base plane
    return _finish("C4", z0 - hh, -hu, -hv, mask, f, f, cx, cy, sigma_deg, rng,
                   {"theta_c_deg": 3.5, "merge_freq": 5})


def config5_map(index: int, size: int = 1024, cells: int = 16) -> Scene:
    """One map of the C5 batch (seed 100 + index)."""
    return voronoi_ortho(f"C5[{index}]", size, size, cells, 100 + index, 0.2)


def config5(count: int = 64, size: int = 1024, cells: int = 16) -> list[Scene]:
    return [config5_map(i, size, cells) for i in range(count)]


CONFIGS = {
    "C1": config1,
    "C2": config2,
    "C3": config3,
    "C4": config4,
}

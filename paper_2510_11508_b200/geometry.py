"""Camera intrinsics and GPU-resident normal / log-depth maps.

Mirrors normint.geometry (geometry.py:31-195): same class names, fields,
validation and error messages, but the arrays live in HBM as torch tensors.
Host numpy views (``.normals``, ``.mask``, ``.values``) are materialised
lazily, so code written against the reference keeps working.

Layout: a map of H x W pixels is stored row-major; normals as float64
structure-of-arrays ``(3, H*W)`` (coalesced per component), validity as one
byte per pixel.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

UNIT_NORM_TOL = 1e-4  # geometry.py:22


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_11508_b200 needs a CUDA device (B200); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


@dataclass(frozen=True)
class CameraIntrinsics:
    """Pinhole intrinsics in pixel units (geometry.py:31-48)."""

    fx: float
    fy: float
    cx: float
    cy: float

    def __post_init__(self):
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError("focal lengths must be positive")
        if not all(np.isfinite([self.fx, self.fy, self.cx, self.cy])):
            raise ValueError("intrinsics must be finite")

    @property
    def mean_focal(self) -> float:
        return 0.5 * (self.fx + self.fy)

    def as_tuple(self):
        return (float(self.fx), float(self.fy), float(self.cx), float(self.cy))


class NormalMap:
    """Unit normals + validity on the GPU (geometry.py:96-153).

    ``batch`` > 1 holds B maps of the same size stacked map-major; the
    kernels never connect pixels of different maps.
    """

    def __init__(self, n_soa: torch.Tensor, valid: torch.Tensor, height: int, width: int,
                 batch: int = 1, valid_count: int | None = None, stats: torch.Tensor | None = None):
        self.n_soa = n_soa  # (3, B*H*W) float64
        self.valid_t = valid  # (B*H*W,) uint8
        self.height = int(height)
        self.width = int(width)
        self.batch = int(batch)
        self._valid_count = valid_count
        self._host_normals = None
        self._host_mask = None

    @property
    def device(self) -> torch.device:
        return self.n_soa.device

    @property
    def npix(self) -> int:
        return self.batch * self.height * self.width

    @property
    def valid_count(self) -> int:
        if self._valid_count is None:
            self._valid_count = int(self.valid_t.sum().item())
        return self._valid_count

    @property
    def normals(self) -> np.ndarray:
        """Host (H, W, 3) float64 view (B, H, W, 3 for a batch), read-only."""
        if self._host_normals is None:
            a = self.n_soa.t().contiguous().cpu().numpy()
            shape = (self.height, self.width, 3) if self.batch == 1 else (
                self.batch, self.height, self.width, 3)
            a = a.reshape(shape)
            a.flags.writeable = False
            self._host_normals = a
        return self._host_normals

    @property
    def mask(self) -> np.ndarray:
        if self._host_mask is None:
            a = self.valid_t.bool().cpu().numpy()
            shape = (self.height, self.width) if self.batch == 1 else (
                self.batch, self.height, self.width)
            a = a.reshape(shape)
            a.flags.writeable = False
            self._host_mask = a
        return self._host_mask

    @classmethod
    def create(cls, normals, mask=None, device=None) -> "NormalMap":
        """Validate and renormalise on the GPU (geometry.py:115-145).

        ``normals``: (H, W, 3) or (B, H, W, 3) array/tensor, float32 or
        float64 (other dtypes are converted to float64 like the reference).
        The float64 norm sqrt((x0^2 + x1^2) + x2^2) and the division are
        IEEE-exact, so the result is bit-identical to numpy's.
        """
        dev = _device(device)
        t = normals if isinstance(normals, torch.Tensor) else torch.from_numpy(np.asarray(normals))
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if t.dim() == 3:
            batch = 1
            h, w = t.shape[0], t.shape[1]
        elif t.dim() == 4:
            batch, h, w = t.shape[0], t.shape[1], t.shape[2]
        else:
            raise ValueError("normals must have shape (H, W, 3)")
        if t.shape[-1] != 3:
            raise ValueError("normals must have shape (H, W, 3)")
        t = t.to(dev).contiguous()
        if mask is None:
            m = None
        else:
            mt = mask if isinstance(mask, torch.Tensor) else torch.from_numpy(np.asarray(mask, dtype=bool))
            if tuple(mt.shape) != tuple(t.shape[:-1]):
                raise ValueError("mask shape does not match normals")
            m = mt.to(dev).to(torch.uint8).contiguous()
        npix = batch * h * w
        from . import devmem
        n_soa = devmem.empty((3, npix), torch.float64, dev)
        valid = devmem.empty(npix, torch.uint8, dev)
        stats = torch.zeros(6, dtype=torch.int64, device=dev)
        lib = _lib.load()
        st = lib.ni_normalize(C.c_void_p(t.data_ptr()), 0 if t.dtype == torch.float32 else 1,
                              C.c_void_p(m.data_ptr() if m is not None else 0), batch, h, w,
                              C.c_void_p(n_soa.data_ptr()), C.c_void_p(valid.data_ptr()),
                              C.c_void_p(stats.data_ptr()), C.c_void_p(_stream(dev)))
        if st == _lib.NI_ERR_EMPTY_MASK:
            # the reference builds an empty map and raises EmptyMask later, in
            # build_pixel_graph (graph.py:65-66); keep that ordering
            return cls(n_soa, valid, h, w, batch, 0)
        _lib.check(st, "NormalMap.create")
        return cls(n_soa, valid, h, w, batch, int(stats[0].item()))

    @classmethod
    def from_unit(cls, normals, mask, device=None) -> "NormalMap":
        """Upload normals that a reference ``NormalMap.create`` already
        validated and renormalised, bit for bit (no second renormalisation:
        n / |n| of a float64 unit vector can move its last bit)."""
        dev = _device(device)
        n = np.asarray(normals, dtype=np.float64)
        m = np.asarray(mask, dtype=bool)
        if n.ndim != 3 or n.shape[2] != 3 or m.shape != n.shape[:2]:
            raise ValueError("normals must have shape (H, W, 3) and mask (H, W)")
        h, w = m.shape
        n_soa = torch.from_numpy(np.ascontiguousarray(n.reshape(-1, 3).T)).to(dev)
        valid = torch.from_numpy(m.reshape(-1).astype(np.uint8)).to(dev)
        n_soa = torch.where(valid.bool()[None, :], n_soa, torch.zeros((), dtype=torch.float64,
                                                                       device=dev))
        return cls(n_soa.contiguous(), valid, h, w, 1, int(m.sum()))

    def flipped(self) -> "NormalMap":
        """All valid normals negated (geometry.py:147-152)."""
        n = torch.where(self.valid_t.bool()[None, :], -self.n_soa, torch.zeros_like(self.n_soa))
        return NormalMap(n, self.valid_t, self.height, self.width, self.batch, self._valid_count)

    def map(self, m: int) -> "NormalMap":
        """Map ``m`` of a batch as a single map (views, no copy)."""
        hw = self.height * self.width
        return NormalMap(self.n_soa[:, m * hw:(m + 1) * hw], self.valid_t[m * hw:(m + 1) * hw],
                         self.height, self.width, 1)


def as_normal_map(nmap, device=None) -> NormalMap:
    """This package's NormalMap, or a reference ``normint.NormalMap`` (any
    object with ``.normals`` (H, W, 3) and ``.mask`` (H, W), geometry.py:96-113)
    uploaded as is."""
    if isinstance(nmap, NormalMap):
        return nmap
    if hasattr(nmap, "normals") and hasattr(nmap, "mask"):
        return NormalMap.from_unit(nmap.normals, nmap.mask, device)
    raise TypeError(f"expected a NormalMap, got {type(nmap).__name__}")


def as_intrinsics(intr) -> CameraIntrinsics:
    """This package's CameraIntrinsics, or any object with fx, fy, cx, cy
    (a reference ``normint.CameraIntrinsics``, geometry.py:31-48)."""
    if isinstance(intr, CameraIntrinsics):
        return intr
    return CameraIntrinsics(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy))


def stack(maps: list[NormalMap]) -> NormalMap:
    """Stack single maps of equal size into one batch (map-major)."""
    if not maps:
        raise ValueError("need at least one map")
    h, w = maps[0].height, maps[0].width
    for m in maps:
        if (m.height, m.width, m.batch) != (h, w, 1):
            raise ValueError("batched maps must share their size")
    n = torch.cat([m.n_soa for m in maps], dim=1).contiguous()
    v = torch.cat([m.valid_t for m in maps]).contiguous()
    return NormalMap(n, v, h, w, len(maps))


class LogDepthMap:
    """Per-pixel natural-log depth sharing the normal map's mask
    (geometry.py:156-177).  ``values_t`` is the float64 device tensor."""

    def __init__(self, values_t: torch.Tensor, mask_t: torch.Tensor, height: int, width: int):
        self.values_t = values_t  # (H*W,) float64, 0 outside the mask
        self.mask_t = mask_t
        self.height = height
        self.width = width
        self._values = None
        self._mask = None

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            a = self.values_t.cpu().numpy().reshape(self.height, self.width)
            a.flags.writeable = False
            self._values = a
        return self._values

    @property
    def mask(self) -> np.ndarray:
        if self._mask is None:
            a = self.mask_t.bool().cpu().numpy().reshape(self.height, self.width)
            a.flags.writeable = False
            self._mask = a
        return self._mask

    def shifted(self, offset: float) -> "LogDepthMap":
        v = torch.where(self.mask_t.bool(), self.values_t + offset, torch.zeros_like(self.values_t))
        return LogDepthMap(v, self.mask_t, self.height, self.width)


def depth_from_logdepth(zmap: LogDepthMap) -> np.ndarray:
    """exp of the log-depth, 0 outside the mask (geometry.py:180-184)."""
    d = torch.where(zmap.mask_t.bool(), torch.exp(zmap.values_t), torch.zeros_like(zmap.values_t))
    return d.cpu().numpy().reshape(zmap.height, zmap.width)

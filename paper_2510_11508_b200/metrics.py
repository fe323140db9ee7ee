"""Depth-map evaluation on the GPU (mirrors normint/metrics.py:1-113).

``evaluate`` aligns the prediction by the median depth ratio and reports MADE
and the relative error; ``min_theoretical_made`` grants every component its
exactly L1-optimal scale.  Both run in libnormint_b200.so (ni_evaluate,
ni_min_theoretical_made) and accept numpy arrays or torch tensors; the
``*_batch`` forms take B stacked maps.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import NoOverlap
from .geometry import _stream


@dataclass(frozen=True)
class EvalReport:
    made: float  # mean absolute depth error after scale alignment
    relative_error: float  # mean |error| / ground-truth depth
    aligned_scale: float  # multiplicative factor applied to the prediction
    valid_pixel_count: int

    def to_dict(self) -> dict:
        return {"made": self.made, "relative_error": self.relative_error,
                "aligned_scale": self.aligned_scale, "valid_pixel_count": self.valid_pixel_count}


def _dev(x, dtype, device):
    t = torch.as_tensor(x)
    return t.to(device=device, dtype=dtype).contiguous()


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("the metrics run on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def evaluate_batch(pred, gt, mask=None) -> list[EvalReport]:
    """``evaluate`` for B stacked maps (B, H, W)."""
    dev = _device()
    p = _dev(pred, torch.float64, dev)
    g = _dev(gt, torch.float64, dev)
    if p.shape != g.shape:
        raise ValueError("prediction and ground truth shapes differ")
    if p.dim() == 2:
        p, g = p[None], g[None]
    B, H, W = p.shape
    m = None if mask is None else _dev(mask, torch.uint8, dev).reshape(B, H, W)
    lib = _lib.load()
    out = torch.empty(4 * B, dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.size_query(lib.ni_evaluate_workspace_size, B, H, W), dtype=torch.uint8,
                     device=dev)
    _lib.check(lib.ni_evaluate(_ptr(p), _ptr(g), _ptr(m), B, H, W, _ptr(out), _ptr(ws),
                               ws.numel(), C.c_void_p(_stream(dev))), "evaluate")
    o = out.cpu().numpy().reshape(B, 4)
    reps = []
    for row in o:
        if row[3] == 0:
            raise NoOverlap("no jointly valid pixel between prediction and ground truth")
        reps.append(EvalReport(float(row[0]), float(row[1]), float(row[2]), int(row[3])))
    return reps


def evaluate(pred, gt, mask=None) -> EvalReport:
    """Median-ratio-aligned depth errors over jointly valid pixels (metrics.py:44-65)."""
    if np.ndim(pred) != 2:
        raise ValueError("evaluate takes one (H, W) map; use evaluate_batch")
    return evaluate_batch(pred, gt, mask)[0]


def min_theoretical_made_batch(pred_depth, gt_depth, labels, map_first, mask=None) -> list[float]:
    """Per-map minimum theoretical MADE.  ``labels``: the batch partition's
    global labels (B, H, W) with map m owning [map_first[m], map_first[m+1])."""
    dev = _device()
    p = _dev(pred_depth, torch.float64, dev)
    g = _dev(gt_depth, torch.float64, dev)
    if p.dim() == 2:
        p, g = p[None], g[None]
    B, H, W = p.shape
    lab = _dev(labels, torch.int32, dev).reshape(B, H, W)
    m = None if mask is None else _dev(mask, torch.uint8, dev).reshape(B, H, W)
    first = np.ascontiguousarray(map_first, dtype=np.int32)
    lib = _lib.load()
    out = torch.empty(2 * B, dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.size_query(lib.ni_min_theoretical_made_workspace_size, B, H, W),
                     dtype=torch.uint8, device=dev)
    _lib.check(lib.ni_min_theoretical_made(_ptr(p), _ptr(g), _ptr(m), _ptr(lab),
                                           C.c_void_p(first.ctypes.data), B, H, W, _ptr(out),
                                           _ptr(ws), ws.numel(), C.c_void_p(_stream(dev))),
               "min_theoretical_made")
    o = out.cpu().numpy().reshape(B, 2)
    if (o[:, 1] == 0).any():
        raise NoOverlap("no jointly valid pixel in any component")
    return [float(v) for v in o[:, 0]]


def min_theoretical_made(pred_depth, gt_depth, partition, mask=None) -> float:
    """Pixel-count-weighted mean of per-component scale-optimal depth errors
    (metrics.py:87-113); ``partition`` is a Partition (labels of the map)."""
    h, w = np.shape(pred_depth)
    base = int(getattr(partition, "label_base", 0))
    labels = getattr(partition, "labels_t", None)
    if labels is None:
        labels = torch.as_tensor(np.asarray(partition.labels))
    return min_theoretical_made_batch(pred_depth, gt_depth, torch.as_tensor(labels).reshape(h, w),
                                      [base, base + partition.component_count], mask)[0]


def l1_optimal_scale(pred, gt) -> float:
    """Scale s minimising sum |s pred - gt| (metrics.py:68-84): the weighted
    median ratio, as one component of ni_min_theoretical_made would pick it."""
    p = np.asarray(pred, np.float64).ravel()
    g = np.asarray(gt, np.float64).ravel()
    if len(p) == 0:
        raise ValueError("need at least one sample")
    dev = _device()
    pt = torch.as_tensor(p, device=dev)
    gtt = torch.as_tensor(g, device=dev)
    ratios = gtt / pt
    order = torch.sort(ratios, stable=True).indices
    w = pt[order].cpu().numpy()
    cum = np.cumsum(w)  # sequential f64 sum, exactly as the reference
    idx = int(np.searchsorted(cum, 0.5 * cum[-1], side="left"))
    return float(ratios[order][idx].item())

"""B200-native drop-in for the component-based normal-integration hot path
of arXiv 2510.11508 (reference package ``normint``).

Public API mirrors normint/__init__.py:3-53 for the hot path:
``run_pipeline`` with ``NormalMap`` / ``CameraIntrinsics`` / ``SolveSettings``
/ ``WeightParams`` in, ``PipelineResult`` out.  All data-parallel work runs in
the sm_100a library ``libnormint_b200.so`` (C ABI: include/normint_b200.h);
there is no CPU fallback.
"""

from .errors import (DegenerateEdge, DeviceError, EmptyMask, NoInterEdges, NormintError)
from .geometry import CameraIntrinsics, LogDepthMap, NormalMap, depth_from_logdepth, stack
from .pipeline import (BaselineResult, Partition, PipelineResult, dot_cutoff, run_pipeline,
                       run_pipeline_batch, run_pipeline_stream, run_pixel_baseline,
                       run_pixel_baseline_batch)
from .seams import (EdgeCoefficients, PixelGraph, QuotientGraph, ScaleStep, apply_scales,
                    build_edge_coefficients, build_pixel_graph, build_quotient, fill_components,
                    form_components, merge_components, relative_scale_step)
from .settings import SolveSettings, WeightParams

__version__ = "0.1.0"

__all__ = [
    "BaselineResult",
    "EdgeCoefficients",
    "PixelGraph",
    "QuotientGraph",
    "ScaleStep",
    "apply_scales",
    "build_edge_coefficients",
    "build_pixel_graph",
    "build_quotient",
    "fill_components",
    "form_components",
    "merge_components",
    "relative_scale_step",
    "CameraIntrinsics",
    "DegenerateEdge",
    "DeviceError",
    "EmptyMask",
    "LogDepthMap",
    "NoInterEdges",
    "NormalMap",
    "NormintError",
    "Partition",
    "PipelineResult",
    "SolveSettings",
    "WeightParams",
    "depth_from_logdepth",
    "dot_cutoff",
    "run_pipeline",
    "run_pipeline_batch",
    "run_pipeline_stream",
    "run_pixel_baseline",
    "run_pixel_baseline_batch",
    "stack",
]

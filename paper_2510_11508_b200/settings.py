"""Run parameters, mirroring the reference's frozen dataclasses.

``SolveSettings`` follows solver.py:26-49 and ``WeightParams`` follows
continuity.py:42-57 (same fields, defaults and validation).  ``worker_count``
is accepted for drop-in compatibility; the GPU solves all components in one
batched launch, so it has no effect.
"""

from __future__ import annotations

from dataclasses import dataclass

CONTINUITY_MODELS = ("milano", "bini")
REWEIGHTING_MODES = ("off", "soft", "hard")


@dataclass(frozen=True)
class SolveSettings:
    cg_tol: float = 1e-6
    cg_max_iters: int = 5000
    delta_e_max: float = 1e-3
    max_iters: int = 150
    alignment_iters: int = 2
    freq_merging: int | None = None
    worker_count: int = 4
    refill_reweighted: bool = False

    def __post_init__(self):
        if not self.cg_tol > 0:
            raise ValueError("cg_tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.alignment_iters < 0:
            raise ValueError("alignment_iters must be non-negative")
        if self.freq_merging is not None and self.freq_merging < 1:
            raise ValueError("freq_merging must be at least 1 when set")
        if self.worker_count < 1:
            raise ValueError("worker_count must be at least 1")


@dataclass(frozen=True)
class WeightParams:
    k: float = 2.0
    outlier_low: float = 1e-5
    outlier_high: float = 1e-3
    reweighting_mode: str = "soft"

    def __post_init__(self):
        if not self.k > 0:
            raise ValueError("k must be positive")
        if not 0 < self.outlier_low < self.outlier_high:
            raise ValueError("need 0 < outlier_low < outlier_high")
        if self.reweighting_mode not in REWEIGHTING_MODES:
            raise ValueError(f"unknown reweighting mode {self.reweighting_mode!r}")

    @property
    def mode_code(self) -> int:
        return REWEIGHTING_MODES.index(self.reweighting_mode)


def _coerce(cls, obj):
    if obj is None or isinstance(obj, cls):
        return obj
    from dataclasses import fields
    return cls(**{f.name: getattr(obj, f.name) for f in fields(cls) if hasattr(obj, f.name)})


def as_settings(obj) -> SolveSettings | None:
    """This package's SolveSettings from a reference ``normint.SolveSettings``
    (same field names, solver.py:26-49), or None."""
    return _coerce(SolveSettings, obj)


def as_weights(obj) -> WeightParams | None:
    """This package's WeightParams from a reference ``normint.WeightParams``
    (continuity.py:42-57), or None."""
    return _coerce(WeightParams, obj)

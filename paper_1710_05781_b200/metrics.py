"""Accuracy metric and seeded instances (mirror of disctree.metrics 26-120).

error_report is the acceptance metric of the reference (metrics.py:91-111):
max relative error over targets whose direct value is not negligible and the
sum-normalised average relative error.  It is a host-side metric on two
value arrays, not part of the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_REL_FLOOR = 1e-12  # metrics.py:29


@dataclass(frozen=True)
class ErrorReport:
    max_relative: float
    avg_relative: float
    excluded_targets: int


def _host(a) -> np.ndarray:
    try:
        import torch

        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy().astype(np.float64)
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(a, dtype=np.float64)


def error_report(tree_values, direct_values) -> ErrorReport:
    tv, dv = _host(tree_values), _host(direct_values)
    if tv.shape != dv.shape or tv.ndim != 1:
        raise ValueError(f"value sequences must match in length, got {tv.shape} vs {dv.shape}")
    if len(tv) == 0:
        raise ValueError("value sequences must be nonempty")
    mag = np.abs(dv)
    scale = float(mag.max())
    if scale == 0.0:
        raise ValueError("all-zero reference: relative errors are undefined")
    diff = np.abs(tv - dv)
    keep = mag >= MAX_REL_FLOOR * scale
    return ErrorReport(
        max_relative=float((diff[keep] / mag[keep]).max()),
        avg_relative=float(diff.sum() / mag.sum()),
        excluded_targets=int(len(tv) - keep.sum()),
    )


def random_instance(n: int, seed, interval: tuple[float, float] = (0.0, 1.0)):
    """n charges uniform in ``interval``, strengths U(0, 1) (metrics.py:114-120)."""
    from .charges import from_particles
    from .workloads import random_instance as pairs

    return from_particles(pairs(n, seed, interval))

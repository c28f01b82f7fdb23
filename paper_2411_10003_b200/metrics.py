"""Load-imbalance metrics (reference ``pkg/src/moebal/simulator.py:106-124``).

balance_degree = population standard deviation of a device-load vector H;
rb_ratio = sigma(before) / sigma(after), with inf when balancing reached a
perfectly flat load from a non-flat one and 1.0 when both are flat.  The
MoE layer reports these on the device-produced H (virtual expert-slot rows
and physical ranks) before and after the plan.
"""

from __future__ import annotations

import math

import numpy as np

from .core import ValidationError


def balance_degree(H) -> float:
    h = np.asarray(H, dtype=np.float64)
    if h.size == 0:
        raise ValidationError("H must be non-empty")
    return float(np.std(h))


def rb_ratio(before, after) -> float:
    s_before = balance_degree(before.H)
    s_after = balance_degree(after.H)
    if s_after == 0.0:
        return 1.0 if s_before == 0.0 else math.inf
    return s_before / s_after


def imbalance_summary(H) -> dict:
    """sigma(H), max/mean and the raw extremes of one load vector."""
    h = np.asarray(H, dtype=np.float64)
    mean = float(h.mean()) if h.size else 0.0
    return {
        "sigma": balance_degree(h),
        "max_over_mean": (float(h.max()) / mean) if mean > 0 else 1.0,
        "max": float(h.max()),
        "min": float(h.min()),
    }

"""Gap-safe sphere radius (reference screening.py:11-15).  The sphere test,
the preserved-set compaction and the z update run on the GPU
(csrc/bx_kernels.cuh: k_sphere, k_scan, k_compact, k_gather)."""

import math

from .errors import NegativeGap


def gap_safe_radius(gap, alpha):
    """sqrt(2 gap / alpha); the gap must be clamped first."""
    if gap < 0:
        raise NegativeGap(f"gap {gap:.3e} is negative; clamp before the radius")
    return math.sqrt(2.0 * gap / alpha)

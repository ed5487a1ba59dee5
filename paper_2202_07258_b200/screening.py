"""Gap-safe sphere radius (reference screening.py:11-15) and the screening
bookkeeping of the per-round API (ScreeningState, safe_screen_test,
apply_screening, forward_product: screening.py:18-104, on the GPU in
primitives.py).  Inside ``solve`` the sphere test, the preserved-set
compaction and the z update are device kernels (csrc/bx_kernels.cuh:
k_sphere, k_scan, k_compact, k_gather)."""

import math

from .errors import NegativeGap


def gap_safe_radius(gap, alpha):
    """sqrt(2 gap / alpha); the gap must be clamped first."""
    if gap < 0:
        raise NegativeGap(f"gap {gap:.3e} is negative; clamp before the radius")
    return math.sqrt(2.0 * gap / alpha)


from .primitives import ScreeningState, apply_screening, forward_product, safe_screen_test  # noqa: E402,F401

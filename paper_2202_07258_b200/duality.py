"""Translation vectors (reference duality.py:339-398).

A ``TranslationVector`` carries the interior direction t; A't and the strict
interiority check are computed on the GPU when the solve context is built
(csrc/bx_kernels.cuh: k_colstats).  The setup-time strategies neg-ones,
neg-column, neg-mean-column and custom are supported; solve-linear (a Cholesky
of A'A, duality.py:380-391) is outside the hot-path scope.
"""

import numpy as np

from .errors import DimensionMismatch

GAP_ROUNDOFF = 1e-9
STRATEGIES = ("neg-ones", "neg-column", "neg-mean-column", "custom")


def clamp_gap(gap):
    """duality.py:450-454."""
    from .errors import InternalConsistency
    if gap < -GAP_ROUNDOFF:
        raise InternalConsistency(f"duality gap {gap:.3e} below round-off slack")
    return max(gap, 0.0)


class TranslationVector:
    """Interior direction t of the dual feasible set (validated on the GPU)."""

    def __init__(self, p, t, strategy="custom"):
        t = np.array(t, dtype=float).ravel()
        if t.shape[0] != p.m:
            raise DimensionMismatch(f"t has length {t.shape[0]}, expected {p.m}")
        self.t = t
        self.strategy = strategy


def select_translation_vector(p, strategy="neg-ones", column=None, t=None):
    if strategy == "neg-ones":
        cand = -np.ones(p.m)
    elif strategy == "neg-column":
        if column is None:
            raise ValueError("neg-column strategy needs a column index")
        cand = -np.asarray(p.a_matrix[:, int(column)], dtype=float).copy()
    elif strategy == "neg-mean-column":
        cand = -np.asarray(p.a_matrix, dtype=float).mean(axis=1)
    elif strategy == "custom":
        if t is None:
            raise ValueError("custom strategy needs an explicit t")
        cand = np.asarray(t, dtype=float)
    else:
        raise ValueError(f"unknown strategy {strategy!r}; choose from {STRATEGIES}")
    return TranslationVector(p, cand, strategy=strategy)

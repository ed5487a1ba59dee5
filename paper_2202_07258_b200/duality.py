"""Translation vectors (reference duality.py:26-100).

A ``TranslationVector`` carries the interior direction t and A't.  Like the
reference it validates strict interiority at construction
(max_j a_j't < -strict_tol ||a_j||, else NoInteriorPoint); A't and the column
norms come from the GPU setup pass (csrc/bx_kernels.cuh: k_colstats).

Strategies (duality.py:62-100): neg-ones, neg-column, neg-mean-column,
custom, and solve-linear -- the least-norm solution of A't = -1 through a
Cholesky factorisation of the Gram matrix A'A, formed and factored on the
device (cuBLAS / cuSOLVER through torch: a one-time setup factorisation, not
the iteration).
"""

import numpy as np

from .errors import DimensionMismatch, NoInteriorPoint, SingularGram

GAP_ROUNDOFF = 1e-9
STRATEGIES = ("neg-ones", "neg-column", "neg-mean-column", "solve-linear", "custom")


def clamp_gap(gap):
    """duality.py:152-156."""
    from .errors import InternalConsistency
    if gap < -GAP_ROUNDOFF:
        raise InternalConsistency(f"duality gap {gap:.3e} below round-off slack")
    return max(gap, 0.0)


class TranslationVector:
    """Strictly interior direction of the dual feasible set, with A't cached."""

    def __init__(self, p, t, strategy="custom", strict_tol=1e-10):
        from .driver import column_stats
        t = np.array(t, dtype=float).ravel()
        if t.shape[0] != p.m:
            raise DimensionMismatch(f"t has length {t.shape[0]}, expected {p.m}")
        norms, att = column_stats(p, t)
        if np.any(att >= -strict_tol * norms):
            raise NoInteriorPoint(f"strategy {strategy!r} did not yield a strictly interior t "
                                  f"(max a_j' t = {att.max():.3e})")
        self.t = t
        self.a_t_t = att
        self.strategy = strategy


def _device_matrix(p):
    """A as an (m, n) fp64 CUDA tensor view/copy of the Problem's storage."""
    import torch
    st = p.device_arrays()["a"]          # (n, lda) row-major == column-major A
    return st[:, : p.m].to(torch.float64).T  # (m, n)


def _solve_linear(p):
    """Least-norm t with A't = -1 (duality.py:82-93): t = A (A'A)^-1 (-1)."""
    import torch
    a = _device_matrix(p)
    b = -torch.ones(p.n, 1, dtype=torch.float64, device=a.device)
    gram = a.T @ a
    chol, info = torch.linalg.cholesky_ex(gram)
    # LAPACK's potrf (the reference's cho_factor) stops at a pivot <= 0; the
    # device factorisation can leave a round-off-sized positive pivot on an
    # exactly rank-deficient Gram matrix (duplicated column) and then solve
    # the consistent system by luck, so a pivot at round-off level relative to
    # the diagonal counts as singular too (rank(A) = n is the requirement)
    if int(info) != 0 or float(torch.diagonal(chol).min()) ** 2 <= 1e-13 * float(torch.diagonal(gram).max()):
        raise SingularGram("A' A is singular; solve-linear needs rank(A) = n <= m")
    cand = a @ torch.cholesky_solve(b, chol)
    # a near-singular Gram matrix can still factor: check the solve itself
    resid = a.T @ cand
    if not torch.allclose(resid, b, rtol=1e-5, atol=1e-6):  # b = -1: atol 1e-6 max(1, |b|)
        raise SingularGram("A' t = b could not be solved accurately")
    return cand.ravel().cpu().numpy()


def select_translation_vector(p, strategy="neg-ones", column=None, t=None):
    """Interior translation vector by one of the reference's recipes."""
    if strategy == "neg-ones":
        cand = -np.ones(p.m)
    elif strategy == "neg-column":
        if column is None:
            raise ValueError("neg-column strategy needs a column index")
        if p.a_matrix is not None:
            cand = -np.asarray(p.a_matrix[:, int(column)], dtype=float).copy()
        else:
            cand = -_device_matrix(p)[:, int(column)].cpu().numpy()
    elif strategy == "neg-mean-column":
        if p.a_matrix is not None:
            cand = -np.asarray(p.a_matrix, dtype=float).mean(axis=1)
        else:
            cand = -_device_matrix(p).mean(dim=1).cpu().numpy()
    elif strategy == "solve-linear":
        cand = _solve_linear(p)
    elif strategy == "custom":
        if t is None:
            raise ValueError("custom strategy needs an explicit t")
        cand = np.asarray(t, dtype=float)
    else:
        raise ValueError(f"unknown strategy {strategy!r}; choose from {STRATEGIES}")
    return TranslationVector(p, cand, strategy=strategy)


# the dual-point family of the per-round API (duality.py:29-209), on the GPU
from .primitives import (DualState, dual_point_bvlr, dual_point_nnlr, dual_translate,  # noqa: E402,F401
                         duality_gap, eval_dual, is_dual_feasible)

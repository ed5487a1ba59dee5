"""Solver configuration and the power-iteration step rule.

Mirrors /root/reference/pkg/src/boxscreen/solvers.py:17-98.  The primal
updates themselves (pg_step :101-116, cd_sweep :119-137, and the FISTA
extension) run on the GPU inside ``bx_solve`` (csrc/bx_core.cu); this module
only carries the configuration and the host side of the step-size rule.
"""

from dataclasses import dataclass

import numpy as np

# "apg" = accelerated projected gradient (FISTA + function-value restart),
# BASELINE.json configs 3 and 5; "active-set" is the reference's third kind
# (bounded Lawson-Hanson, solvers.py:140-204; csrc/bx_active.cuh).
_SOLVER_KINDS = ("pg", "cd", "apg", "active-set")


@dataclass
class SolverConfig:
    kind: str = "cd"
    step_size: float | None = None  # None = auto via power iteration
    power_iters: int = 50
    inner_passes: int = 1
    max_rounds: int | None = None
    gap_tol: float = 1e-6
    # stop on gap <= gap_tol * max(1, P) instead of gap <= gap_tol; None = the
    # reference's absolute rule for fp64, the relative rule for fp32 storage
    # (an absolute 1e-6 is below fp32 resolution when P* >> 1)
    relative_gap: bool | None = None
    # FISTA ("apg") restart rule: "adaptive" restarts on an objective increase
    # or on the O'Donoghue-Candes gradient test (the default);
    # "function" restarts on an objective increase only -- BASELINE config 3's
    # stated rule (the objective-rise test of solvers.py:111-114)
    restart: str = "adaptive"

    def __post_init__(self):
        if self.kind not in _SOLVER_KINDS:
            raise ValueError(f"unknown solver kind {self.kind!r}")
        if self.gap_tol <= 0:
            raise ValueError("gap_tol must be positive")
        if self.restart not in ("adaptive", "function"):
            raise ValueError(f"unknown restart rule {self.restart!r}")
        if self.inner_passes < 1:
            raise ValueError("inner_passes must be >= 1")


def start_vector(k, seed=0):
    """Power-iteration start: default_rng(seed).standard_normal(k), normalised
    (solvers.py:75-77).  Host-side numpy, handed to the native loop through a
    callback so the GPU step size matches the reference's to rounding."""
    v = np.random.default_rng(seed).standard_normal(k)
    v /= np.linalg.norm(v)
    return v


def spectral_norm_estimate(a_sub, power_iters=50, seed=0):
    """Largest singular value by power iteration on A'A, run on the GPU
    (solvers.py:72-86).  ``a_sub`` is host (numpy) or a CUDA tensor."""
    from .driver import _Session
    from .model import Problem
    a = a_sub
    n = a.shape[1]
    p = Problem(a, np.zeros(a.shape[0]), np.zeros(n), np.ones(n))
    with _Session(p) as s:
        return s.power_iter(power_iters, start_vector(n, seed))


def auto_step_size(a_sub, alpha, power_iters=50):
    """0.99 alpha / (sigma/0.999)^2 (solvers.py:89-98)."""
    sigma = spectral_norm_estimate(a_sub, power_iters=power_iters) / 0.999
    if sigma == 0.0:
        return 1.0
    return 0.99 * alpha / sigma ** 2


# the spec-level one-shot updates (solvers.py:38-45, 207-240), on the GPU
from .primitives import ActiveSetState, active_set_update, cd_update, pg_update  # noqa: E402,F401

"""Acceptance criteria 7 and 8 of the reference (pkg/tests/test_acceptance.py:
235-296) on the GPU path:

* the certified gap of every converged solve, recomputed from scratch on the
  host with fresh products (no cached residual, norms or dual point), is
  below the tolerance it was certified at;
* the active-set kind reaches the exact optimum of small NNLS problems, as
  found by enumerating all 2^n passive patterns.
"""

import itertools

import numpy as np
import pytest

from conftest import small_instance

pytestmark = pytest.mark.gpu


def test_certified_gap_from_scratch():
    from oracle.boxscreen_oracle import certified_gap
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    rng = np.random.default_rng(3)
    worst, runs = 0.0, 0
    for i in range(40):
        family = ("nnls", "bvls", "mixed")[i % 3]
        kind = ("pg", "cd", "active-set", "apg")[(i // 3) % 4]
        n = int(rng.integers(4, 25))
        m = n + int(rng.integers(0, 30))
        a, y, lo, hi = small_instance(rng, m, n, family)
        res = solve(Problem(a, y, lo, hi), SolverConfig(kind=kind, gap_tol=1e-6, inner_passes=10), screening=True)
        if not res.converged:
            continue
        runs += 1
        a64 = np.ascontiguousarray(a, dtype=np.float64)
        inf_mask = np.isinf(hi)
        t = -np.ones(m)
        gap, _, _, _ = certified_gap(a64, y, lo, hi, inf_mask, np.asarray(res.x, dtype=np.float64), t, a64.T @ t)
        worst = max(worst, gap)
    assert runs >= 35, runs
    assert worst < 1e-6, worst


def _exhaustive_nnls(a, y):
    """min 0.5 ||a x - y||^2 over x >= 0 by enumerating passive sets."""
    n = a.shape[1]
    best = np.inf
    for pattern in itertools.product((0, 1), repeat=n):
        free = [j for j in range(n) if pattern[j]]
        x = np.zeros(n)
        if free:
            x[free] = np.linalg.lstsq(a[:, free], y, rcond=None)[0]
        if np.any(x < 0.0):
            continue
        r = a @ x - y
        best = min(best, 0.5 * float(r @ r))
    return best


def test_active_set_matches_exhaustive_pattern_oracle():
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    rng = np.random.default_rng(21)
    worst = 0.0
    for _ in range(50):
        n = int(rng.integers(2, 9))
        m = n + int(rng.integers(1, 10))
        a, y, lo, hi = small_instance(rng, m, n, "nnls")
        res = solve(Problem(a, y, lo, hi), SolverConfig(kind="active-set"), screening=False)
        r = a @ res.x - y
        obj = 0.5 * float(r @ r)
        best = _exhaustive_nnls(np.asarray(a), y)
        worst = max(worst, abs(obj - best) / max(1.0, best))
    assert worst <= 1e-8, worst

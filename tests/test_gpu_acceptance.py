"""Acceptance-style safety and equivalence on many random instances, after the
reference's criteria 1 and 2 (pkg/tests/test_acceptance.py:33-100): every
screened coordinate is saturated in a high-accuracy solution, and screening
on/off reach the same objective."""

import itertools

import numpy as np
import pytest

from conftest import small_instance

pytestmark = pytest.mark.gpu


def _cases(count=216, seed=20240817):
    # the reference's 216 instances over nnls / bvls / mixed x pg / cd /
    # active-set, plus the apg kind
    rng = np.random.default_rng(seed)
    combos = list(itertools.product(("nnls", "bvls", "mixed"), ("pg", "apg", "cd", "active-set")))
    for i in range(count):
        family, kind = combos[i % len(combos)]
        n = int(rng.integers(3, 31))
        m = int(rng.integers(n, 61))
        yield (family, kind) + small_instance(rng, m, n, family)


def test_criterion1_screening_is_safe_and_criterion2_on_off_agree():
    from oracle.boxscreen_oracle import oracle_solve
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    checked = violations = 0
    worst = 0.0
    for family, kind, a, y, lo, hi in _cases():
        p = Problem(a, y, lo, hi)
        cfg = SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-8)
        on = solve(p, cfg, screening=True)
        off = solve(p, cfg, screening=False)
        assert on.converged and off.converged, (family, kind)
        # high-accuracy reference point: the CPU oracle's FISTA to a 1e-12 gap
        ref = oracle_solve(a, y, lo, hi, kind="apg", inner_passes=10, gap_tol=1e-12, max_rounds=50000,
                           screening=False)
        for j in on.sat_lower:
            checked += 1
            violations += abs(ref["x"][j] - lo[j]) >= 1e-7
        for j in on.sat_upper:
            checked += 1
            violations += abs(ref["x"][j] - hi[j]) >= 1e-7
        o_on = 0.5 * float(np.sum((a @ on.x - y) ** 2))
        o_off = 0.5 * float(np.sum((a @ off.x - y) ** 2))
        worst = max(worst, abs(o_on - o_off) / max(1.0, abs(o_off)))
    assert checked > 200
    assert violations == 0, f"{violations} of {checked} screened coordinates not saturated"
    assert worst <= 1e-8, worst

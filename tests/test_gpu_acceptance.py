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


def test_criterion3_translation_validity_and_fixed_point():
    """Reference criterion 3 (pkg/tests/test_acceptance.py:103-125, Prop. 1):
    the translated point is dual feasible for every z, and a feasible z is a
    fixed point, exactly.  A'z and the scaling run on the device."""
    from paper_2202_07258_b200 import Problem, dual_translate, select_translation_vector
    rng = np.random.default_rng(7)
    worst = -np.inf
    for _ in range(300):
        m, n = (int(v) for v in rng.integers(2, 15, 2))
        a, y, lo, hi = small_instance(rng, m, n, "nnls")
        p = Problem(a, y, lo, hi)
        tv = select_translation_vector(p, "neg-ones")
        out = dual_translate(p, tv, rng.standard_normal(m) * 3.0)
        worst = max(worst, float((a.T @ out).max()))
    assert worst <= 1e-12, worst
    fixed = 0
    for _ in range(100):
        m, n = (int(v) for v in rng.integers(2, 15, 2))
        a, y, lo, hi = small_instance(rng, m, n, "nnls")
        p = Problem(a, y, lo, hi)
        tv = select_translation_vector(p, "neg-ones")
        z = -np.abs(rng.standard_normal(m))
        if np.any(a.T @ z > 0.0):
            continue
        out = dual_translate(p, tv, z)
        assert (out == z).all()
        fixed += 1
    assert fixed > 50


def test_criterion4_four_matrix_classes():
    """Reference criterion 4 (test_acceptance.py:128-172, Prop. 2): each matrix
    class has its interior translation vector (A't < 0 from the device's
    column statistics), and a rank-deficient Gram matrix is refused."""
    from paper_2202_07258_b200 import Problem, select_translation_vector
    from paper_2202_07258_b200.errors import NoInteriorPoint, SingularGram
    rng = np.random.default_rng(11)
    per_class = {"solve-linear": 0, "orthogonal": 0, "neg-ones": 0, "neg-column": 0}
    trials = 25
    for _ in range(trials):
        n = int(rng.integers(2, 8))
        m = n + int(rng.integers(0, 8))
        a = rng.standard_normal((m, n))
        tv = select_translation_vector(Problem(a, np.zeros(m), 0.0, np.inf), "solve-linear")
        per_class["solve-linear"] += int(np.all(tv.a_t_t < 0))
        q, _ = np.linalg.qr(rng.standard_normal((m, n)))
        coeff = rng.uniform(0.5, 2.0, n)
        tv = select_translation_vector(Problem(q, np.zeros(m), 0.0, np.inf), "custom", t=-(q @ coeff))
        per_class["orthogonal"] += int(np.all(tv.a_t_t < 0))
        a, y, lo, hi = small_instance(rng, m, n, "nnls")
        p = Problem(a, y, lo, hi)
        per_class["neg-ones"] += int(np.all(select_translation_vector(p, "neg-ones").a_t_t < 0))
        j = int(rng.integers(n))
        per_class["neg-column"] += int(np.all(select_translation_vector(p, "neg-column", column=j).a_t_t < 0))
    assert all(v == trials for v in per_class.values()), per_class
    a = rng.standard_normal((6, 3))
    p_bad = Problem(np.column_stack([a, a[:, 0]]), np.zeros(6), 0.0, np.inf)
    with pytest.raises((SingularGram, NoInteriorPoint)):
        select_translation_vector(p_bad, "solve-linear")


def test_criterion9_numerical_units():
    """Reference criterion 9 (test_acceptance.py:299-337): Fenchel-Young
    inequality of the loss pair, the gradient against finite differences, the
    device power iteration against the SVD, and the screened forward product
    against the dense product."""
    from paper_2202_07258_b200 import (PrimalPoint, Problem, ScreeningState, apply_screening, conj_loss, eval_loss,
                                       forward_product, grad_loss, spectral_norm_estimate)
    rng = np.random.default_rng(33)
    z, u, y = (rng.uniform(-10, 10, 10 ** 4) for _ in range(3))
    assert float(np.min(eval_loss(z, y) + conj_loss(u, y) - z * u)) >= -1e-12
    h = 1e-5
    for _ in range(200):
        zz, yy = rng.uniform(-10, 10, 2)
        fd = (eval_loss(zz + h, yy) - eval_loss(zz - h, yy)) / (2 * h)
        assert abs(grad_loss(zz, yy) - fd) < 1e-6
    for _ in range(10):
        a = rng.standard_normal((20, 10))
        true = np.linalg.svd(a, compute_uv=False)[0]
        assert abs(spectral_norm_estimate(a) - true) / true < 1e-3
    for _ in range(20):
        a, yv, lo, hi = small_instance(rng, 6, 10, "bvls")
        p = Problem(a, yv, lo, hi)
        st = ScreeningState(p)
        pt = PrimalPoint(np.clip(np.zeros(10), lo, hi))
        apply_screening(st, np.array([1, 3]), np.array([5]), pt, p)
        x_full = pt.x.copy()
        x_full[st.preserved] = rng.uniform(lo[st.preserved], hi[st.preserved])
        got = forward_product(st, p, x_full[st.preserved])
        np.testing.assert_allclose(got, a @ x_full, rtol=1e-10, atol=1e-12)

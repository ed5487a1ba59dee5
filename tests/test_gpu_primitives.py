"""The per-round API on the GPU.

1. The spec-level primitives the reference exports next to ``solve``
   (/root/reference/pkg/src/boxscreen/__init__.py:3-16) against the
   reference's own outputs on the same inputs (tests/golden/primitives.npz,
   made by tests/golden/make_golden.py from the unmodified reference):
   pg_update / cd_update / active_set_update, dual_point_nnlr / _bvlr,
   eval_dual, is_dual_feasible, duality_gap, dual_translate,
   safe_screen_test, apply_screening, forward_product.
2. The fine-grained C ABI (bx_primal_passes, bx_dual_screen,
   bx_certified_gap, bx_compact, bx_get_state, bx_power_iter) stepping
   Algorithm 1's rounds by hand (driver.py:168-241) against the oracle, round
   by round, for PG and FISTA.
"""

import ctypes
import os

import numpy as np
import pytest

from conftest import small_instance
from oracle.boxscreen_oracle import oracle_solve
from parity import OBJ_RTOL

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "primitives.npz"))
CASES = sorted({k.split("/")[0] for k in GOLD.files})


def g(case, name):
    return GOLD[f"{case}/{name}"]


def close(a, b, rtol=1e-9, atol=1e-12):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = max(1.0, float(np.max(np.abs(b))) if b.size else 1.0)
    d = float(np.max(np.abs(a - b))) if a.size else 0.0
    assert d <= rtol * scale + atol, (d, scale)


@pytest.mark.parametrize("case", CASES)
def test_spec_level_sequence_matches_reference(case):
    import paper_2202_07258_b200 as bx
    a, y, lo, hi = g(case, "a"), g(case, "y"), g(case, "lo"), g(case, "hi")
    p = bx.Problem(a, y, lo, hi)
    st = bx.ScreeningState(p)
    close(st.col_norms, np.linalg.norm(a, axis=0), 1e-14)
    pt = bx.PrimalPoint(np.clip(np.zeros(p.n), lo, hi))
    step = float(g(case, "step"))
    r1, g1 = bx.pg_update(p, st, pt, bx.SolverConfig(kind="pg", inner_passes=3000), step)
    close(pt.x, g(case, "pg_x"))
    close(r1, g(case, "pg_r"))
    close(g1, g(case, "pg_g"))
    # dual point of the reference's iterate (so the rest compares like with like)
    pt.x = g(case, "pg_x").copy()
    pt.ax_cache = None
    if p.j_inf.size:
        tv = bx.select_translation_vector(p, "neg-ones")
        ds = bx.dual_point_nnlr(p, tv, pt)
        close(bx.dual_translate(p, tv, g(case, "zgrad")), g(case, "translated"))
    else:
        ds = bx.dual_point_bvlr(p, pt)
    scale = max(abs(float(g(case, "d_value"))), 1.0)
    close(ds.theta, g(case, "theta"))
    close(ds.a_t_theta_cache, g(case, "a_t_theta"))
    assert abs(ds.d_value - float(g(case, "d_value"))) <= OBJ_RTOL * scale
    assert abs(ds.gap - float(g(case, "gap"))) <= OBJ_RTOL * scale
    theta = g(case, "theta")
    assert abs(bx.eval_dual(p, theta) - float(g(case, "eval_dual"))) <= OBJ_RTOL * scale
    assert abs(bx.eval_dual(p, theta, g(case, "a_t_theta")) - float(g(case, "eval_dual_cached"))) <= OBJ_RTOL * scale
    assert bx.is_dual_feasible(p, theta) == bool(g(case, "feasible"))
    assert bx.is_dual_feasible(p, -theta) == bool(g(case, "feasible_neg"))
    assert abs(bx.duality_gap(p, pt, theta) - float(g(case, "duality_gap"))) <= OBJ_RTOL * scale
    # sphere tests: the reference's decisions on its own dual point, and on a
    # synthetic vector with decisions on both sides
    st.radius = float(g(case, "radius"))
    nl, nu = bx.safe_screen_test(st, g(case, "a_t_theta"), p, slack=float(g(case, "slack")))
    np.testing.assert_array_equal(nl, g(case, "new_lower"))
    np.testing.assert_array_equal(nu, g(case, "new_upper"))
    st.radius = 0.5
    nl2, nu2 = bx.safe_screen_test(st, g(case, "vtest"), p, slack=0.25)
    np.testing.assert_array_equal(nl2, g(case, "new_lower2"))
    np.testing.assert_array_equal(nu2, g(case, "new_upper2"))
    st.radius = float(g(case, "radius"))
    bx.apply_screening(st, nl, nu, pt, p)
    close(st.z, g(case, "z"))
    np.testing.assert_array_equal(st.preserved, g(case, "preserved"))
    close(pt.x, g(case, "x_screened"), 0.0, 0.0)
    close(bx.forward_product(st, p, pt.x[st.preserved]), g(case, "forward"))
    r2, g2 = bx.cd_update(p, st, pt, bx.SolverConfig(kind="cd", inner_passes=3))
    close(pt.x, g(case, "cd_x"))
    close(r2, g(case, "cd_r"))
    close(g2, g(case, "cd_g"))
    # active set from the reference's start
    st3 = bx.ScreeningState(p)
    pt3 = bx.PrimalPoint(lo.copy())
    ass = bx.ActiveSetState(p.n)
    for it in range(3):
        r3, g3, opt = bx.active_set_update(p, st3, pt3, ass, bx.SolverConfig(kind="active-set"))
        np.testing.assert_array_equal(ass.passive, g(case, f"as{it}_passive"))
        assert opt == bool(g(case, f"as{it}_opt"))
        close(pt3.x, g(case, f"as{it}_x"), 1e-8)
        close(r3, g(case, f"as{it}_r"), 1e-8)
        close(g3, g(case, f"as{it}_g"), 1e-8)


def test_primitive_errors_like_the_reference():
    import paper_2202_07258_b200 as bx
    from paper_2202_07258_b200 import errors as E
    rng = np.random.default_rng(5)
    a, y, lo, hi = small_instance(rng, 20, 10, "nnls")
    p = bx.Problem(a, y, lo, hi)
    pt = bx.PrimalPoint(np.zeros(10))
    with pytest.raises(E.WrongVariant):
        bx.dual_point_bvlr(p, pt)
    with pytest.raises(E.DimensionMismatch):
        bx.eval_dual(p, np.zeros(3))
    st = bx.ScreeningState(p)
    with pytest.raises(E.IndexOutOfPreserved):
        bx.apply_screening(st, np.array([3]), np.array([], int), pt, p)
        bx.apply_screening(st, np.array([3]), np.array([], int), pt, p)
    with pytest.raises(E.InfeasiblePoint):
        bx.eval_primal(p, bx.PrimalPoint(-np.ones(10)))
    with pytest.raises(E.DualInfeasible):
        bx.duality_gap(p, pt, np.asarray(y) * 1e6)


def test_eval_primal_uncached_on_gpu():
    """model.py:109-120 with A x formed on the GPU."""
    import paper_2202_07258_b200 as bx
    p = bx.Problem(np.eye(2), [1.0, 1.0], 0.0, 2.0)
    assert bx.eval_primal(p, bx.PrimalPoint([1.0, 1.0])) == 0.0
    assert bx.eval_primal(p, bx.PrimalPoint([0.0, 1.0])) == 0.5
    rng = np.random.default_rng(12345)
    for _ in range(10):
        m, n = (int(v) for v in rng.integers(1, 12, 2))
        a, y = rng.standard_normal((m, n)), rng.standard_normal(m)
        q = bx.Problem(a, y, -2.0, 2.0)
        x = rng.uniform(-2, 2, n)
        plain, cached = bx.eval_primal(q, bx.PrimalPoint(x)), bx.eval_primal(q, bx.PrimalPoint(x, ax_cache=a @ x))
        assert abs(plain - cached) <= 1e-10 * max(1.0, abs(plain))


# ---------------------------------------------------------------------------
# Algorithm 1 stepped through the fine-grained C ABI
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("family", ["nnls", "bvls", "mixed"])
@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_rounds_through_fine_grained_abi(family, kind, monkeypatch):
    """driver.py:168-241 written as calls of the C ABI: primal passes, dual
    point + sphere test, certified gap when the reduced gap is below the
    tolerance, compaction, step re-estimate when the preserved set halves --
    every round's P, D, gap and preserved count against the oracle, and the
    final x / screened sets through bx_get_state."""
    import torch
    from oracle.boxscreen_oracle import safe_step
    from paper_2202_07258_b200 import Problem
    from paper_2202_07258_b200 import _native as nat
    from paper_2202_07258_b200.driver import _Session
    from paper_2202_07258_b200.solvers import start_vector
    monkeypatch.setenv("BX_NO_SMALL", "1")
    rng = np.random.default_rng(77 + ["nnls", "bvls", "mixed"].index(family))
    a, y, lo, hi = small_instance(rng, 120, 300, family)
    # FISTA amplifies round-off differences between any two summation orders
    # (~10x per 10 rounds on these instances, PG stays at 1e-14:
    # profiles/r02_fista_roundoff_drift.txt), so its per-round 1e-10 check
    # covers the first 40 rounds
    passes, tol, rounds = 10, 1e-9, (80 if kind == "pg" else 40)
    o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=passes, gap_tol=tol, max_rounds=rounds)
    L = nat.lib()
    s = _Session(Problem(a, y, lo, hi))
    try:
        ctx = s.ctx
        nat.check(L.bx_reset(ctx), ctx, "bx_reset")

        def power():
            sig = ctypes.c_double()
            k = L.bx_preserved_count(ctx)
            v0 = np.ascontiguousarray(start_vector(k))
            nat.check(L.bx_power_iter(ctx, 50, v0.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      ctypes.byref(sig)), ctx, "bx_power_iter")
            sg = sig.value / 0.999
            return 1.0 if sg == 0.0 else 0.99 / sg ** 2

        eta = power()
        assert abs(eta - safe_step(a)) <= 1e-12 * eta
        basis = a.shape[1]
        out = (ctypes.c_double * 8)()
        cert = (ctypes.c_double * 4)()
        n_done = 0
        for rnd in range(1, len(o["trace"]) + 1):
            nat.check(L.bx_primal_passes(ctx, nat.KINDS[kind], eta, passes), ctx, "bx_primal_passes")
            nat.check(L.bx_dual_screen(ctx, 1, 1e-12, 1.0, out), ctx, "bx_dual_screen")
            ot = o["trace"][rnd - 1]
            sc = max(abs(ot["primal"]), abs(ot["dual"]), 1e-3)
            for i, key in enumerate(("primal", "dual", "gap")):
                assert abs(out[i] - ot[key]) <= OBJ_RTOL * sc, (rnd, key, out[i], ot[key])
            assert int(out[6]) == ot["new_lower"] and int(out[7]) == ot["new_upper"], rnd
            if out[2] < tol:
                nat.check(L.bx_certified_gap(ctx, 1.0, cert), ctx, "bx_certified_gap")
                if ot["certified"] is not None:
                    assert abs(cert[0] - ot["certified"]) <= OBJ_RTOL * sc
            nat.check(L.bx_compact(ctx), ctx, "bx_compact")
            k = L.bx_preserved_count(ctx)
            assert k == ot["preserved"], rnd
            if k < 0.5 * basis:
                eta = power()
                basis = k
            n_done = rnd
            if ot["certified"] is not None and ot["certified"] < tol:
                break
        assert n_done == len(o["trace"])
        n = a.shape[1]
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        sl = torch.empty(max(len(o["sat_lower"]), 1), dtype=torch.int64, device="cuda")
        su = torch.empty(max(len(o["sat_upper"]), 1), dtype=torch.int64, device="cuda")
        nat.check(L.bx_get_state(ctx, x.data_ptr(), None, sl.data_ptr(), su.data_ptr()), ctx, "bx_get_state")
        xo = o["x"]
        assert float(np.max(np.abs(x.cpu().numpy() - xo))) <= 1e-8 * max(1.0, float(np.max(np.abs(xo))))
        np.testing.assert_array_equal(np.sort(sl.cpu().numpy()[: len(o["sat_lower"])]), np.sort(o["sat_lower"]))
        np.testing.assert_array_equal(np.sort(su.cpu().numpy()[: len(o["sat_upper"])]), np.sort(o["sat_upper"]))
    finally:
        s.close()

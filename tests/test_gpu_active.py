"""The active-set kind (bounded Lawson-Hanson, reference solvers.py:140-204)
on the GPU against the REAL reference's outputs (tests/golden/active_cases.npz,
cfg1_as_trace.npz from make_golden.py) and against the oracle.

The device path keeps the passive Cholesky factor across iterations (column
appends, Givens deletions; csrc/bx_active.cuh) where the reference refactors
it each time, so the iterates agree to rounding, not bit for bit: the
north_star tolerances apply (objective / gap 1e-10 relative, x 1e-8).
"""

import os

import numpy as np
import pytest

from parity import OBJ_RTOL, X_RTOL, compare_final, compare_traces

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def _inputs(z, key):
    if str(z[key + "_meta"][0]) == "medium":
        from conftest import medium_nnls
        return medium_nnls()
    return z[key + "_a"], z[key + "_y"], z[key + "_lo"], z[key + "_hi"]


def _check(res, z, key):
    pfx = key + "_tr_"
    tr = res.trace
    assert len(tr) == len(z[pfx + "primal"]), f"{key} rounds gpu={len(tr)} ref={len(z[pfx + 'primal'])}"
    rp, rd, rg, rk = (z[pfx + f] for f in ("primal", "dual", "gap", "preserved"))
    scale = np.maximum(np.maximum(np.abs(rp), np.abs(rd)), 1e-3)
    for name, ref in (("primal", rp), ("dual", rd), ("gap", rg)):
        got = np.array([getattr(t, name) for t in tr])
        bad = np.flatnonzero(np.abs(got - ref) > OBJ_RTOL * scale)
        assert bad.size == 0, f"{key} {name}: round {bad[0] + 1} gpu={got[bad[0]]!r} ref={ref[bad[0]]!r}"
    np.testing.assert_array_equal([t.preserved_count for t in tr], rk, err_msg=key)
    x_ref = z[key + "_x"]
    den = max(1.0, float(np.max(np.abs(x_ref))))
    assert float(np.max(np.abs(res.x - x_ref))) / den <= X_RTOL, key
    np.testing.assert_array_equal(np.sort(res.sat_lower), np.sort(z[key + "_sat_lower"]), err_msg=key)
    np.testing.assert_array_equal(np.sort(res.sat_upper), np.sort(z[key + "_sat_upper"]), err_msg=key)
    gap, rounds, conv = z[key + "_final"]
    assert res.converged == bool(conv) and res.rounds == int(rounds), key
    assert abs(res.gap - gap) <= OBJ_RTOL * max(1.0, abs(float(rp[-1]))), key


def test_active_cases_vs_reference():
    """nnls / bvls / mixed x screening on/off, the reference suite's KATs and
    a 300 x 600 screened NNLS instance (compaction rebuilds the factor)."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    z = _load("active_cases.npz")
    for i in range(int(z["count"])):
        key = f"c{i:03d}"
        fam, _, scr = (str(v) for v in z[key + "_meta"])
        a, y, lo, hi = _inputs(z, key)
        tol = 1e-6 if fam == "kat" else 1e-8
        res = solve(Problem(a, y, lo, hi), SolverConfig(kind="active-set", gap_tol=tol), screening=scr == "1")
        _check(res, z, key)


def test_kat_two_iteration_and_immediate_optimality():
    """test_solvers.py:144-159: x = [1, 0] after two outer iterations; w <= 0
    at x = 0 means nothing enters and the first round is optimal."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    res = solve(Problem(np.eye(2), [1.0, -1.0], 0.0, np.inf), SolverConfig(kind="active-set"), screening=False)
    np.testing.assert_allclose(res.x, [1.0, 0.0], atol=1e-12)
    assert res.converged
    res = solve(Problem(np.eye(2), [-1.0, -2.0], 0.0, np.inf), SolverConfig(kind="active-set"), screening=False)
    np.testing.assert_allclose(res.x, [0.0, 0.0])
    assert res.rounds == 1 and res.converged


def test_cfg1_instance_full_trajectory():
    """BASELINE config 1's instance (1000 x 2000 NNLS) through the active-set
    kind: all 287 rounds against the reference's own run; up to ~280 passive
    columns in the factor, screening compactions in between."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    z = _load("cfg1_as_trace.npz")
    inst = make_config(1)
    res = solve(Problem(inst.a, inst.y, inst.lower, inst.upper), SolverConfig(kind="active-set", gap_tol=1e-6))
    tr = res.trace
    rp, rd, rg, rk = (z["tr_" + f] for f in ("primal", "dual", "gap", "preserved"))
    assert len(tr) == len(rp)
    scale = np.maximum(np.maximum(np.abs(rp), np.abs(rd)), 1e-3)
    for name, ref in (("primal", rp), ("dual", rd), ("gap", rg)):
        got = np.array([getattr(t, name) for t in tr])
        bad = np.flatnonzero(np.abs(got - ref) > OBJ_RTOL * scale)
        assert bad.size == 0, f"{name}: round {bad[0] + 1} gpu={got[bad[0]]!r} ref={ref[bad[0]]!r}"
    np.testing.assert_array_equal([t.preserved_count for t in tr], rk)
    den = max(1.0, float(np.max(np.abs(z["x"]))))
    assert float(np.max(np.abs(res.x - z["x"]))) / den <= X_RTOL
    np.testing.assert_array_equal(np.sort(res.sat_lower), np.sort(z["sat_lower"]))
    assert res.converged


@pytest.mark.parametrize("family", ["nnls", "bvls", "mixed"])
def test_vs_oracle_and_solvers_agree(family):
    """Against the oracle round by round, and the three reference kinds reach
    the same objective (test_solvers.py:179-205)."""
    from conftest import small_instance
    from oracle.boxscreen_oracle import objective, oracle_solve
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    rng = np.random.default_rng(9090 + len(family))
    a, y, lo, hi = small_instance(rng, 70, 45, family)
    p = Problem(a, y, lo, hi)
    res = solve(p, SolverConfig(kind="active-set", gap_tol=1e-10), screening=True)
    orc = oracle_solve(a, y, lo, hi, kind="active-set", gap_tol=1e-10, screening=True)
    assert not compare_traces(res, orc)
    assert not compare_final(res, orc)
    ref = objective(a, y, res.x)
    for kind in ("pg", "cd"):
        other = solve(p, SolverConfig(kind=kind, gap_tol=1e-10, inner_passes=20), screening=False)
        assert other.converged
        assert abs(objective(a, y, other.x) - ref) <= 1e-7 * max(1.0, abs(ref)), kind


def test_fp32_storage():
    """fp32 A: same optimum as fp64 within the fp32 objective tolerance."""
    from conftest import medium_nnls
    from oracle.boxscreen_oracle import objective
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    a, y, lo, hi = medium_nnls()
    r64 = solve(Problem(a, y, lo, hi), SolverConfig(kind="active-set", gap_tol=1e-8))
    r32 = solve(Problem(a, y, lo, hi, dtype=np.float32), SolverConfig(kind="active-set", gap_tol=1e-6))
    o64, o32 = objective(a, y, r64.x), objective(a.astype(np.float32).astype(float), y, r32.x)
    assert abs(o32 - o64) <= 1e-4 * max(1.0, o64)

"""The CPU oracle pinned against the REAL reference's outputs (golden fixtures
made by tests/golden/make_golden.py from /root/reference).  CPU only."""

import os

import numpy as np
import pytest

from oracle.boxscreen_oracle import OracleError, certified_gap, column_norms, oracle_solve, spectral_sigma

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return np.load(path, allow_pickle=False)


def _cases(z):
    for i in range(int(z["count"])):
        key = f"c{i:03d}"
        fam, kind, scr = (str(v) for v in z[key + "_meta"])
        yield key, fam, kind, scr == "1"


def test_small_cases_bitwise():
    """pg and cd, nnls/bvls/mixed, screening on/off: every trace value equal."""
    z = _load("small_cases.npz")
    n_checked = 0
    for key, fam, kind, scr in _cases(z):
        o = oracle_solve(z[key + "_a"], z[key + "_y"], z[key + "_lo"], z[key + "_hi"], kind=kind,
                         inner_passes=10, gap_tol=1e-8, screening=scr)
        gap, rounds, conv = z[key + "_final"]
        assert o["rounds"] == int(rounds), key
        assert o["converged"] == bool(conv), key
        assert o["gap"] == gap, key
        for f, ref in (("primal", "primal"), ("dual", "dual"), ("gap", "gap"), ("preserved", "preserved")):
            got = np.array([r[f] for r in o["trace"]])
            np.testing.assert_array_equal(got, z[f"{key}_tr_{ref}"], err_msg=f"{key} {f}")
        np.testing.assert_array_equal(o["x"], z[key + "_x"], err_msg=key)
        np.testing.assert_array_equal(o["theta"], z[key + "_theta"], err_msg=key)
        np.testing.assert_array_equal(o["sat_lower"], z[key + "_sat_lower"])
        np.testing.assert_array_equal(o["sat_upper"], z[key + "_sat_upper"])
        n_checked += 1
    assert n_checked == 36


def test_kat_cases():
    z = _load("kat_cases.npz")
    for name in z["names"]:
        name = str(name)
        step = float(z[name + "_step"])
        o = oracle_solve(z[name + "_a"], z[name + "_y"], z[name + "_lo"], z[name + "_hi"],
                         kind=str(z[name + "_kind"]), inner_passes=int(z[name + "_passes"]), gap_tol=1e-6,
                         step_size=None if np.isnan(step) else step)
        np.testing.assert_array_equal(o["x"], z[name + "_x"], err_msg=name)
        gap, rounds, conv = z[name + "_final"]
        assert o["rounds"] == int(rounds) and o["converged"] == bool(conv), name


def test_cfg1_prefix_bitwise():
    """BASELINE config 1 at full size: the oracle reproduces the reference's
    first 150 rounds (1500 PG steps) exactly."""
    from paper_2202_07258_b200.generate import make_config
    z = _load("cfg1_trace.npz")
    inst = make_config(1)
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind="pg", inner_passes=10, gap_tol=1e-6,
                     max_rounds=150)
    for f in ("primal", "dual", "gap", "preserved"):
        got = np.array([r[f] for r in o["trace"]])
        np.testing.assert_array_equal(got, z["tr_" + f][:150], err_msg=f)


def test_cfg2_prefix_bitwise():
    """BASELINE config 2 (CD, BVLS) at full size: first 15 sweeps exactly."""
    from paper_2202_07258_b200.generate import make_config
    z = _load("cfg2_trace.npz")
    inst = make_config(2)
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind="cd", inner_passes=1, gap_tol=1e-7,
                     max_rounds=15)
    for f in ("primal", "dual", "gap", "preserved"):
        got = np.array([r[f] for r in o["trace"]])
        np.testing.assert_array_equal(got, z["tr_" + f][:15], err_msg=f)


def _active_inputs(z, key):
    if str(z[key + "_meta"][0]) == "medium":
        import hashlib
        from conftest import medium_nnls
        a, y, lo, hi = medium_nnls()
        h = hashlib.sha256()
        for arr in (a, y):
            h.update(np.ascontiguousarray(arr).tobytes())
        assert h.hexdigest() == str(z[key + "_digest"])
        return a, y, lo, hi
    return z[key + "_a"], z[key + "_y"], z[key + "_lo"], z[key + "_hi"]


def test_active_set_cases_bitwise():
    """The active-set kind (bounded Lawson-Hanson, solvers.py:140-204):
    every trace value, the final state and the saturated sets equal."""
    z = _load("active_cases.npz")
    n_checked = 0
    for key, fam, kind, scr in _cases(z):
        a, y, lo, hi = _active_inputs(z, key)
        tol = 1e-6 if fam == "kat" else 1e-8
        o = oracle_solve(a, y, lo, hi, kind="active-set", gap_tol=tol, screening=scr)
        gap, rounds, conv = z[key + "_final"]
        assert (o["rounds"], o["converged"], o["gap"]) == (int(rounds), bool(conv), gap), key
        for f in ("primal", "dual", "gap", "preserved"):
            got = np.array([r[f] for r in o["trace"]])
            np.testing.assert_array_equal(got, z[f"{key}_tr_{f}"], err_msg=f"{key} {f}")
        np.testing.assert_array_equal(o["x"], z[key + "_x"], err_msg=key)
        np.testing.assert_array_equal(o["theta"], z[key + "_theta"], err_msg=key)
        np.testing.assert_array_equal(o["sat_lower"], z[key + "_sat_lower"])
        np.testing.assert_array_equal(o["sat_upper"], z[key + "_sat_upper"])
        n_checked += 1
    assert n_checked == 21
    # test_solvers.py:144-147: the two-iteration example lands on [1, 0]
    np.testing.assert_allclose(z["c018_x"], [1.0, 0.0], atol=1e-12)


def test_cfg1_active_set_prefix_bitwise():
    """BASELINE config 1's instance through the active-set kind: the first 60
    outer iterations exactly (the full 287 take ~5 s more)."""
    from paper_2202_07258_b200.generate import make_config
    z = _load("cfg1_as_trace.npz")
    inst = make_config(1)
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind="active-set", gap_tol=1e-6, max_rounds=60)
    for f in ("primal", "dual", "gap", "preserved"):
        got = np.array([r[f] for r in o["trace"]])
        np.testing.assert_array_equal(got, z["tr_" + f][:60], err_msg=f)


def test_apg_solution_level_pin():
    """The FISTA extension is not in the reference: pinned at solution level
    against the reference's active-set optimum (certified gap 1e-12): objective
    within the cross-solver tolerance (test_solvers.py:205) and every screened
    coordinate saturated in the optimum (test_acceptance.py:69-88)."""
    z = _load("optimum_cases.npz")
    for key in z["names"]:
        key = str(key)
        a, y, lo, hi = z[key + "_a"], z[key + "_y"], z[key + "_lo"], z[key + "_hi"]
        o = oracle_solve(a, y, lo, hi, kind="apg", inner_passes=10, gap_tol=1e-10)
        assert o["converged"], key
        r = a @ o["x"] - y
        obj = 0.5 * float(r @ r)
        ref = float(z[key + "_obj"])
        assert abs(obj - ref) <= 1e-7 * max(1.0, abs(ref)), key
        xs = z[key + "_x"]
        for j in o["sat_lower"]:
            assert abs(xs[j] - lo[j]) < 1e-7, (key, j)
        for j in o["sat_upper"]:
            assert abs(xs[j] - hi[j]) < 1e-7, (key, j)


def test_oracle_errors_and_units():
    with pytest.raises(OracleError) as e:
        oracle_solve(np.array([[1.0, 0.0], [1.0, 0.0]]), np.zeros(2), 0.0, np.inf)
    assert e.value.kind == "NoInteriorPoint"
    with pytest.raises(OracleError) as e:
        oracle_solve(np.array([[1.0, 0.0], [1.0, 0.0]]), np.zeros(2), 0.0, 1.0)
    assert e.value.kind == "ZeroColumn"
    assert spectral_sigma(np.eye(3)) == pytest.approx(1.0, abs=1e-6)
    assert spectral_sigma(np.diag([3.0, 1.0])) == pytest.approx(3.0, abs=1e-4)
    np.testing.assert_allclose(column_norms(np.array([[3.0, 0.0], [4.0, 2.0]])), [5.0, 2.0])
    # certified gap at the 1-D optimum is zero (test_duality.py:261-264)
    gap, theta, p, d = certified_gap(np.array([[1.0]]), np.array([-1.0]), np.zeros(1), np.full(1, np.inf),
                                     np.array([True]), np.zeros(1), -np.ones(1), np.array([-1.0]))
    assert gap == pytest.approx(0.0, abs=1e-12)

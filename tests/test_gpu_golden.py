"""GPU vs the REAL reference: the CUDA path through the C ABI compared with the
reference package's own outputs (golden fixtures generated from
/root/reference by tests/golden/make_golden.py), including BASELINE configs 1
and 2 at full size, round by round."""

import os

import numpy as np
import pytest

from parity import OBJ_RTOL, X_RTOL

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def _check_trace(res, z, prefix="tr_", key=""):
    tr = res.trace
    n = min(len(tr), len(z[prefix + "primal"]))
    gp = np.array([t.primal for t in tr[:n]])
    gd = np.array([t.dual for t in tr[:n]])
    gg = np.array([t.gap for t in tr[:n]])
    gk = np.array([t.preserved_count for t in tr[:n]])
    rp, rd, rg, rk = (z[prefix + f][:n] for f in ("primal", "dual", "gap", "preserved"))
    scale = np.maximum(np.maximum(np.abs(rp), np.abs(rd)), 1e-3)
    for name, a, b in (("primal", gp, rp), ("dual", gd, rd), ("gap", gg, rg)):
        bad = np.flatnonzero(np.abs(a - b) > OBJ_RTOL * scale)
        assert bad.size == 0, f"{key} {name}: first bad round {bad[0] + 1}: gpu={a[bad[0]]!r} ref={b[bad[0]]!r}"
    bad = np.flatnonzero(gk != rk)
    assert bad.size == 0, f"{key} preserved: first bad round {bad[0] + 1}: gpu={gk[bad[0]]} ref={rk[bad[0]]}"
    assert len(tr) == len(z[prefix + "primal"]), f"{key} rounds gpu={len(tr)} ref={len(z[prefix + 'primal'])}"


def _check_final(res, x_ref, sl, su, key=""):
    den = max(1.0, float(np.max(np.abs(x_ref))))
    assert float(np.max(np.abs(res.x - x_ref))) / den <= X_RTOL, key
    np.testing.assert_array_equal(np.sort(res.sat_lower), np.sort(sl), err_msg=key)
    np.testing.assert_array_equal(np.sort(res.sat_upper), np.sort(su), err_msg=key)


def test_small_cases_vs_reference():
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    z = _load("small_cases.npz")
    for i in range(int(z["count"])):
        key = f"c{i:03d}"
        fam, kind, scr = (str(v) for v in z[key + "_meta"])
        p = Problem(z[key + "_a"], z[key + "_y"], z[key + "_lo"], z[key + "_hi"])
        res = solve(p, SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-8), screening=scr == "1")
        _check_trace(res, z, prefix=key + "_tr_", key=key)
        _check_final(res, z[key + "_x"], z[key + "_sat_lower"], z[key + "_sat_upper"], key)
        gap, rounds, conv = z[key + "_final"]
        assert res.converged == bool(conv) and res.rounds == int(rounds), key


def test_kat_cases_vs_reference():
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    z = _load("kat_cases.npz")
    for name in z["names"]:
        name = str(name)
        step = float(z[name + "_step"])
        p = Problem(z[name + "_a"], z[name + "_y"], z[name + "_lo"], z[name + "_hi"])
        res = solve(p, SolverConfig(kind=str(z[name + "_kind"]), inner_passes=int(z[name + "_passes"]),
                                    gap_tol=1e-6, step_size=None if np.isnan(step) else step))
        np.testing.assert_allclose(res.x, z[name + "_x"], rtol=0, atol=1e-14, err_msg=name)
        gap, rounds, conv = z[name + "_final"]
        assert res.rounds == int(rounds) and res.converged == bool(conv), name
        assert res.trace[-1].screening_ratio == float(z[name + "_ratio"]), name


@pytest.mark.parametrize("streamed", [False, True])
@pytest.mark.parametrize("cfg_id,fname", [(1, "cfg1_trace.npz"), (2, "cfg2_trace.npz")])
def test_baseline_config_full_trajectory(cfg_id, fname, streamed, monkeypatch):
    """BASELINE config 1 (PG, 24k rounds) and 2 (CD) at full size: every round's
    primal / dual / gap / preserved count against the reference's own run."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    if streamed:
        if cfg_id == 2:
            pytest.skip("CD has one path")
        monkeypatch.setenv("BX_NO_SMALL", "1")   # force the streamed k_pass path
    z = _load(fname)
    inst = make_config(cfg_id)
    res = solve(Problem(inst.a, inst.y, inst.lower, inst.upper),
                SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol))
    _check_trace(res, z, key=f"cfg{cfg_id}")
    _check_final(res, z["x"], z["sat_lower"], z["sat_upper"], key=f"cfg{cfg_id}")
    assert res.converged

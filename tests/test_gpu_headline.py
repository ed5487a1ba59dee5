"""Round-by-round oracle parity for the headline path at its own shapes.

The fused streamed pass is instantiated per row-chunk count R (rows per
thread = R 16-byte vectors, csrc/bx_core.cu pick_R); BASELINE config 3
(m = 10,000) runs the R = 10 fp64 instantiation and config 4 (m = 20,000
fp32) the R = 10 fp32 one.  These tests compare every round of those
instantiations -- and of every R in 6..12 -- with the CPU oracle
(oracle/boxscreen_oracle.py, pinned to the reference): primal, dual and gap
within 1e-10 * max(|P|, |D|) and identical preserved counts every round
(reference round loop: /root/reference/pkg/src/boxscreen/driver.py:168-241).

* R sweep, fp64, two families per m: the config-3 recipe (no screening event
  in the first rounds: pure streaming) and a BVLS saturation family whose
  coordinates leave the preserved set over several rounds (compaction,
  incremental refresh and the speculative round-boundary pass at that R).
* R sweep, fp32 storage, against the fp64 oracle on the same rounded matrix:
  per-round objective within 1e-4 relative (north_star's fp32 tolerance).
* config 3 itself (10000 x 50000, 4 GB): the first 60 rounds against
  ``oracle_solve(max_rounds=60)``.
"""

import numpy as np
import pytest

from oracle.boxscreen_oracle import oracle_solve
from parity import OBJ_RTOL, compare_final, compare_traces

pytestmark = pytest.mark.gpu

# m -> R of the fp64 pass (R = ceil(m / 1024)); ragged and exact multiples
FP64_M = {6: 5121, 7: 6145, 8: 7169, 9: 8193, 10: 10000, 11: 11264, 12: 12288}
# fp32 moves 4 rows per 16-byte vector: R = ceil(m / 2048)
FP32_M = {7: 12289, 9: 16385, 10: 20000, 12: 24576}


def saturating_bvls(m, n, seed):
    """Gaussian unit columns, box [-1, 1], planted solution 40% at +-1.3 (so
    its coordinates saturate and are screened over several rounds)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    a /= np.linalg.norm(a, axis=0)
    xt = rng.choice([-1.3, 1.3, 0.0], size=n, p=[0.4, 0.4, 0.2])
    mid = xt == 0.0
    xt[mid] = rng.uniform(-0.5, 0.5, int(mid.sum()))
    y = a @ xt + 0.01 * rng.standard_normal(m)
    return np.asfortranarray(a), y, -np.ones(n), np.ones(n)


def _solve(a, y, lo, hi, kind, passes, tol, rounds, dtype=np.float64, restart="adaptive"):
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    p = Problem(a, y, lo, hi, dtype=dtype)
    return solve(p, SolverConfig(kind=kind, inner_passes=passes, gap_tol=tol, max_rounds=rounds,
                                 restart=restart))


@pytest.mark.parametrize("R", sorted(FP64_M))
@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_fp64_rsweep_config3_recipe(R, kind, monkeypatch):
    from paper_2202_07258_b200.generate import make_config
    monkeypatch.setenv("BX_NO_SMALL", "1")
    inst = make_config(3, m=FP64_M[R], n=1500)
    g = _solve(inst.a, inst.y, inst.lower, inst.upper, kind, 10, 1e-6, 40)
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind=kind, inner_passes=10, gap_tol=1e-6,
                     max_rounds=40)
    probs = compare_traces(g, o)
    assert not probs, (R, probs[:3])
    assert len(g.trace) == 40


@pytest.mark.parametrize("R", sorted(FP64_M))
@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_fp64_rsweep_screening_events(R, kind, monkeypatch):
    monkeypatch.setenv("BX_NO_SMALL", "1")
    a, y, lo, hi = saturating_bvls(FP64_M[R], 1500, seed=R)
    g = _solve(a, y, lo, hi, kind, 3, 1e-11, 200)
    o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=3, gap_tol=1e-11, max_rounds=200)
    assert sum(r["new_lower"] + r["new_upper"] > 0 for r in o["trace"]) >= 2  # several events
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, (R, probs[:3])


@pytest.mark.parametrize("R", sorted(FP32_M))
@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_fp32_rsweep_tracks_fp64_oracle(R, kind):
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(4, m=FP32_M[R], n=1500)
    assert inst.a.dtype == np.float32
    rounds = 30
    g = _solve(inst.a, inst.y, inst.lower, inst.upper, kind, 10, 1e-6, rounds, dtype=np.float32)
    a64 = np.asfortranarray(inst.a.astype(np.float64))  # the same rounded matrix
    o = oracle_solve(a64, inst.y, inst.lower, inst.upper, kind=kind, inner_passes=10, gap_tol=1e-300,
                     max_rounds=rounds)
    assert len(g.trace) == rounds == len(o["trace"])
    p32 = np.array([t.primal for t in g.trace])
    p64 = np.array([t["primal"] for t in o["trace"]])
    assert np.all(np.abs(p32 - p64) <= 1e-4 * np.abs(p64)), (R, np.max(np.abs(p32 - p64) / np.abs(p64)))


def test_config3_first_60_rounds():
    """BASELINE config 3 at its full size (R = 10 fp64 pass): the first 60
    rounds (600 FISTA steps + 60 dual points) against the oracle."""
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(3)
    assert inst.a.shape == (10000, 50000)
    g = _solve(inst.a, inst.y, inst.lower, inst.upper, "apg", 10, 1e-6, 60)
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind="apg", inner_passes=10, gap_tol=1e-6,
                     max_rounds=60)
    probs = compare_traces(g, o)
    assert not probs, probs[:3]
    assert len(g.trace) == 60


@pytest.mark.parametrize("path", ["resident", "streamed"])
def test_function_restart_rule_matches_oracle(path, monkeypatch):
    """BASELINE config 3's stated FISTA rule -- restart on an objective
    increase only (SolverConfig(restart="function")) -- round by round on the
    config-3 recipe at an oracle-friendly size, both device paths."""
    from paper_2202_07258_b200.generate import make_config
    if path == "streamed":
        monkeypatch.setenv("BX_NO_SMALL", "1")
    else:
        monkeypatch.delenv("BX_NO_SMALL", raising=False)
    inst = make_config(3, m=500, n=2500)
    g = _solve(inst.a, inst.y, inst.lower, inst.upper, "apg", 10, 1e-6, 400, restart="function")
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind="apg", inner_passes=10, gap_tol=1e-6,
                     max_rounds=400, restart="function")
    probs = compare_traces(g, o) + (compare_final(g, o) if o["converged"] else [])
    assert not probs, probs[:3]
    adaptive = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind="apg", inner_passes=10,
                            gap_tol=1e-6, max_rounds=400)
    # the two rules are different iterations (the gradient test fires)
    assert [t["primal"] for t in adaptive["trace"][:50]] != [t["primal"] for t in o["trace"][:50]]


@pytest.fixture(params=["spec", "no_spec", "force_undo"])
def spec_mode(request, monkeypatch):
    """The round boundary's three schedules: the speculative step
    (default), a dot-only screening pass per round (BX_SPEC=0), and every
    screening event undoing the speculative step (BX_SPEC_FORCE_UNDO=1)."""
    monkeypatch.delenv("BX_SPEC", raising=False)
    monkeypatch.delenv("BX_SPEC_FORCE_UNDO", raising=False)
    if request.param == "no_spec":
        monkeypatch.setenv("BX_SPEC", "0")
    elif request.param == "force_undo":
        monkeypatch.setenv("BX_SPEC_FORCE_UNDO", "1")
    return request.param


@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_round_boundary_schedules_match_oracle(kind, spec_mode, monkeypatch):
    """Every round-boundary schedule follows the oracle round by round
    through screening events at both bounds (z updates with nonzero bounds),
    and so does the final x; with the speculative step most events keep it."""
    monkeypatch.setenv("BX_NO_SMALL", "1")
    a, y, lo, hi = saturating_bvls(3000, 900, seed=5)
    g = _solve(a, y, lo, hi, kind, 4, 1e-11, 300)
    o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=4, gap_tol=1e-11, max_rounds=300)
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]
    events = sum(r["new_lower"] + r["new_upper"] > 0 for r in o["trace"])
    assert events >= 3
    if spec_mode == "spec":
        assert g.info["spec_kept"] >= 1
    elif spec_mode == "force_undo":
        assert g.info["spec_kept"] == 0 and g.info["spec_undone"] >= 1
    else:
        assert g.info["spec_kept"] == g.info["spec_undone"] == 0


@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_speculative_step_dropped_at_round_limit(kind, monkeypatch):
    """A solve that stops at max_rounds right after a screening event whose
    speculative step stood: the returned x is the last round's iterate (the
    step is dropped through the compaction that followed it)."""
    monkeypatch.setenv("BX_NO_SMALL", "1")
    a, y, lo, hi = saturating_bvls(2000, 700, seed=9)
    full = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=3, gap_tol=1e-11, max_rounds=60)
    ev = [r["round"] for r in full["trace"] if r["new_lower"] + r["new_upper"] > 0]
    assert len(ev) >= 2
    for rounds in sorted(set(ev[:4] + [e + 1 for e in ev[:2]])):
        g = _solve(a, y, lo, hi, kind, 3, 1e-11, rounds)
        o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=3, gap_tol=1e-11, max_rounds=rounds)
        probs = compare_traces(g, o) + compare_final(g, o)
        assert not probs, (rounds, probs[:3])


def _basis_at(tr, r, n):
    """Preserved count at the last step re-estimate up to round r (1-based):
    the driver re-estimates eta when the preserved set halves
    (driver.py:232-235)."""
    steps = tr["step"][:r]
    ch = np.flatnonzero(steps[1:] != steps[:-1])
    return int(tr["preserved_count"][ch[-1] + 1]) if ch.size else n


def test_config3_screening_events_replayed_from_device_state():
    """Config 3's screening events at full size (10000 x 50000): the device
    solve is stopped just before an event round, the oracle resumes from the
    device's state (x, x_prev, momentum, screened sets, step, basis) and its
    next rounds -- the event round included -- must match the device's round
    by round: P, D, gap within 1e-10 * max(|P|, |D|), identical preserved and
    newly screened counts (replay, since a CPU trajectory to
    the first event takes hours; FISTA also amplifies round-off between any
    two summation orders, profiles/r02_fista_roundoff_drift.txt)."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(3)
    a, y, lo, hi = inst.a, inst.y, inst.lower, inst.upper
    n = a.shape[1]
    p = Problem(a, y, lo, hi)
    cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6)
    full = solve(p, cfg)
    assert full.converged
    tr = full.info["trace_arrays"]
    newly = tr["newly_screened_lower"] + tr["newly_screened_upper"]
    ev = np.flatnonzero(newly > 0) + 1  # event rounds (1-based)
    assert ev.size >= 10
    steps = tr["step"]
    reest = np.flatnonzero(steps[1:] != steps[:-1]) + 2  # rounds that re-estimated eta
    picks = {int(ev[0]), int(ev[len(ev) // 2]), int(ev[-1])}
    if reest.size:
        picks.add(int(reest[0]))
    R = 3
    for e in sorted(picks):
        e = max(e, 2)
        pre = solve(p, SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=e - 1),
                    prev_iterate=True)
        assert pre.rounds == e - 1
        st = dict(x=pre.x, x_prev=pre.info["x_prev"], sat_lower=pre.sat_lower, sat_upper=pre.sat_upper,
                  eta=float(steps[e - 2]), basis=_basis_at(tr, e - 1, n), mom=float(tr["momentum"][e - 2]),
                  round0=e - 1)
        o = oracle_solve(a, y, lo, hi, kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=R, init=st)
        for i, ot in enumerate(o["trace"]):
            gt = full.trace[e - 1 + i]
            assert gt.round == ot["round"] == e + i
            sc = max(abs(ot["primal"]), abs(ot["dual"]))
            for key in ("primal", "dual", "gap"):
                assert abs(getattr(gt, key) - ot[key]) <= OBJ_RTOL * sc, (e + i, key, getattr(gt, key), ot[key])
            assert gt.preserved_count == ot["preserved"], (e + i, gt.preserved_count, ot["preserved"])
            assert gt.newly_screened_lower == ot["new_lower"] and gt.newly_screened_upper == ot["new_upper"], e + i
            if ot.get("certified") is not None and ot["certified"] < 1e-6:
                break


@pytest.mark.parametrize("path", ["streamed", "small"])
@pytest.mark.parametrize("kind,dtype", [("pg", np.float64), ("apg", np.float64), ("pg", np.float32)])
def test_zero_coefficient_skip_is_exact(path, kind, dtype, monkeypatch):
    """The fused step (and the small-round kernel's partial-row loop) skips the
    axpy of a column whose new coefficient is zero.  a_j * 0 adds nothing to a
    partial row, so the trajectory must not change by one bit: every trace
    value, x and theta of a sparse NNLS solve are compared bitwise with the
    skip switched off (BX_NO_ZSKIP, read when the context is created)."""
    from paper_2202_07258_b200.generate import make_config
    if path == "streamed":
        monkeypatch.setenv("BX_NO_SMALL", "1")
    if path == "small" and dtype == np.float32:
        pytest.skip("the small-round kernel is exercised in fp64")
    # config-3 recipe: 2% nonzeros, most of x on its bound; the small size is SM-resident
    m, n = (1537, 3001) if path == "streamed" else (600, 1000)
    inst = make_config(3, m=m, n=n, seed=5)
    rounds = 40
    out = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("BX_NO_ZSKIP", "1")
        else:
            monkeypatch.delenv("BX_NO_ZSKIP", raising=False)
        out.append(_solve(inst.a.astype(dtype), inst.y, inst.lower, inst.upper, kind, 10, 1e-9, rounds, dtype=dtype))
    on, ref = out
    assert on.rounds == ref.rounds and len(on.trace) == len(ref.trace) >= 5
    assert np.count_nonzero(on.x) < on.x.size                # the skip had something to skip
    for r_on, r_ref in zip(on.trace, ref.trace):
        assert r_on.primal == r_ref.primal and r_on.dual == r_ref.dual and r_on.gap == r_ref.gap
        assert r_on.preserved_count == r_ref.preserved_count
    assert np.array_equal(on.x, ref.x) and np.array_equal(on.theta, ref.theta)

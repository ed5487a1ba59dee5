"""Parity at BASELINE's full sizes through size-independent properties
(the per-round oracle comparison runs at reduced sizes elsewhere; a full CPU
trajectory at these sizes takes hours).

* config 3 (10000 x 50000 fp64, 4 GB): the solve's certificate is recomputed
  on the host in fp64 from the returned x alone (oracle.certified_gap, i.e.
  duality.py's dual point and objective) -- the gap must be below the
  tolerance and agree with the device's certified gap; screened coordinates
  sit exactly at their bound.
* config 4 (one 20000 x 62,500 fp32 shard, 5 GB): the fp32-storage PG path
  tracks the fp64 path on the same rounded matrix to 1e-4 relative objective
  on every round (north_star's fp32 tolerance).
* config 5 (K = 100,000 right-hand sides): problems are independent, so a
  seeded sample of 64 of them, run through the batched oracle, must match the
  full-K GPU run problem by problem (primal, dual, gap within 1e-10 of
  max(|P|, |D|); identical preserved counts).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_config3_full_size_independent_certificate():
    from oracle.boxscreen_oracle import certified_gap
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(3)
    a, y = inst.a, inst.y
    res = solve(Problem(a, y, inst.lower, inst.upper),
                SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6))
    assert res.converged and res.gap <= 1e-6, (res.rounds, res.gap)
    x = np.asarray(res.x, dtype=np.float64)
    assert np.all(x >= 0.0)
    # screened coordinates are exactly at the bound (apply_screening snaps them)
    assert res.sat_lower.size > 0.5 * a.shape[1]
    assert np.all(x[res.sat_lower] == 0.0)
    # independent fp64 certificate from x alone (t = -1, A't recomputed here)
    t = -np.ones(a.shape[0])
    att = a.T @ t
    inf_mask = np.isinf(inst.upper)
    gap, _, primal, dual = certified_gap(a, y, inst.lower, inst.upper, inf_mask, x, t=t, att=att)
    scale = max(abs(primal), abs(dual))
    assert gap <= 1e-6 + 1e-10 * scale, gap
    assert abs(gap - res.gap) <= 1e-10 * scale, (gap, res.gap)
    assert abs(primal - res.trace[-1].primal) <= 1e-6 + 1e-10 * scale


def test_config4_full_shard_fp32_tracks_fp64():
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    argv, sys.argv = sys.argv, sys.argv[:1]
    try:
        import bench
    finally:
        sys.argv = argv
    from oracle.boxscreen_oracle import objective
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    inst = bench.make_instance(4)
    assert inst.a.dtype == np.float32 and inst.a.shape == (20000, 62500)
    rounds = 30
    cfg = SolverConfig(kind="pg", inner_passes=10, gap_tol=1e-6, max_rounds=rounds)
    r32 = solve(Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=np.float32), cfg)
    a64 = np.asfortranarray(inst.a, dtype=np.float64)   # the same rounded matrix
    r64 = solve(Problem(a64, inst.y, inst.lower, inst.upper), cfg)
    assert r32.rounds == r64.rounds == rounds
    p32 = np.array([t.primal for t in r32.trace])
    p64 = np.array([t.primal for t in r64.trace])
    assert np.all(np.abs(p32 - p64) <= 1e-4 * np.abs(p64)), np.max(np.abs(p32 - p64) / np.abs(p64))
    # the fp32 run's final iterate, evaluated in fp64
    f32 = objective(a64, inst.y, np.asarray(r32.x, dtype=np.float64))
    f64 = objective(a64, inst.y, np.asarray(r64.x, dtype=np.float64))
    assert abs(f32 - f64) <= 1e-4 * abs(f64), (f32, f64)


def test_config5_full_K_sample_matches_batched_oracle():
    from oracle.batched_oracle import batched_apg
    from paper_2202_07258_b200.batched import solve_batched
    from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
    a = bump_dictionary(200, 5000)
    Y, _ = batched_rhs(a, 100000)
    g = solve_batched(a, Y, passes=10, rounds=2, gap_tol=1e-300)
    assert g.rounds == 2 and g.x.shape == (5000, 100000)
    idx = np.sort(np.random.default_rng(7).choice(100000, size=64, replace=False))
    o = batched_apg(a, np.ascontiguousarray(Y[:, idx]), eta=g.eta, inner_passes=10, rounds=2, gap_tol=1e-300)
    scale = np.maximum(np.maximum(np.abs(o["primal"][-1]), np.abs(o["dual"][-1])), 1e-3)
    for name, gv in (("primal", g.primal), ("dual", g.dual), ("gap", g.gap)):
        d = np.abs(gv[idx] - o[name][-1])
        assert np.all(d <= 1e-10 * scale), (name, d.max())
    np.testing.assert_array_equal(g.preserved[idx], o["preserved"][-1])
    assert np.max(np.abs(g.x[:, idx] - o["X"])) <= 1e-8 * max(1.0, np.abs(o["X"]).max())


def test_config4_full_shard_fp32_against_fp64_oracle():
    """Config 4's full 20000 x 62,500 fp32 shard against the fp64 oracle
    directly (not only through the fp64 device path): the first 10 rounds'
    objectives within north_star's 1e-4 relative fp32 tolerance."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    argv, sys.argv = sys.argv, sys.argv[:1]
    try:
        import bench
    finally:
        sys.argv = argv
    from oracle.boxscreen_oracle import oracle_solve
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    inst = bench.make_instance(4)
    rounds = 10
    r32 = solve(Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=np.float32),
                SolverConfig(kind="pg", inner_passes=10, gap_tol=1e-6, max_rounds=rounds))
    a64 = np.asfortranarray(inst.a, dtype=np.float64)  # the same rounded matrix
    o = oracle_solve(a64, inst.y, inst.lower, inst.upper, kind="pg", inner_passes=10, gap_tol=1e-300,
                     max_rounds=rounds)
    p32 = np.array([t.primal for t in r32.trace])
    p64 = np.array([t["primal"] for t in o["trace"]])
    assert p32.shape == p64.shape == (rounds,)
    assert np.all(np.abs(p32 - p64) <= 1e-4 * np.abs(p64)), np.max(np.abs(p32 - p64) / np.abs(p64))

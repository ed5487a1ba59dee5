"""Edge shapes of every device path vs the oracle, round by round: ragged row
counts (odd m, m % 4 != 0 for the fp32 16-byte vectors), single rows and
columns, the small-path / streamed-path / register-envelope boundaries, and
a problem whose whole preserved set is screened away (k = 0 afterwards)."""

import numpy as np
import pytest

from oracle.boxscreen_oracle import objective, oracle_solve
from parity import compare_final, compare_traces
from test_gpu_parity import _solve_both

pytestmark = pytest.mark.gpu


def _nnls(m, n, seed):
    rng = np.random.default_rng(seed)
    a = np.abs(rng.standard_normal((m, n))) + 0.05
    y = a @ (np.maximum(rng.standard_normal(n), 0.0) * (rng.random(n) < 0.3)) + 0.05 * rng.standard_normal(m)
    return np.asfortranarray(a), y, np.zeros(n), np.full(n, np.inf)


@pytest.mark.parametrize("m,n", [(1, 5), (3, 1), (7, 40), (1001, 300), (4096, 300), (4097, 300)])
@pytest.mark.parametrize("kind", ["pg", "apg", "cd"])
@pytest.mark.parametrize("streamed", [False, True])
def test_ragged_and_boundary_shapes(m, n, kind, streamed, monkeypatch):
    if streamed:
        monkeypatch.setenv("BX_NO_SMALL", "1")
    else:
        monkeypatch.delenv("BX_NO_SMALL", raising=False)
    a, y, lo, hi = _nnls(m, n, seed=m * 31 + n)
    g, o = _solve_both(a, y, lo, hi, kind, passes=10 if kind != "cd" else 1, tol=1e-9, max_rounds=30)
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]


@pytest.mark.parametrize("kind", ["pg", "apg", "cd"])
def test_everything_screened(kind):
    """A >= 0 and y < 0: x* = 0 and every column is screened within a few
    rounds; the rounds after that run on an empty preserved set."""
    rng = np.random.default_rng(11)
    a = np.asfortranarray(np.abs(rng.standard_normal((50, 80))) + 0.1)
    y = -np.abs(rng.standard_normal(50)) - 0.5
    g, o = _solve_both(a, y, np.zeros(80), np.full(80, np.inf), kind, passes=10, tol=1e-10, max_rounds=50)
    assert g.converged and o["converged"]
    assert g.trace[-1].preserved_count == 0 and len(g.sat_lower) == 80
    np.testing.assert_array_equal(g.x, 0.0)
    assert not compare_traces(g, o)


@pytest.mark.parametrize("m", [5, 1023, 4099])
def test_fp32_ragged_rows(m):
    """fp32 storage moves 4 rows per 16-byte vector: ragged m exercises the
    guarded last vector of the dot and the unguarded axpy padding."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    a, y, lo, hi = _nnls(m, 200, seed=m)
    a32 = np.asfortranarray(a.astype(np.float32))
    res = solve(Problem(a32, y, lo, hi, dtype=np.float32),
                SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=20000))
    # converged: certified by the fp64-accumulated certificate (the reduced
    # gap of the fp32-accumulated residual has a floor)
    assert res.converged, (res.rounds, res.gap)
    ref = oracle_solve(np.asfortranarray(a32.astype(np.float64)), y, lo, hi, kind="apg", inner_passes=10,
                       gap_tol=1e-9 * max(1.0, float(res.trace[-1].primal)))
    p32 = objective(a32.astype(np.float64), y, np.asarray(res.x, dtype=np.float64))
    p64 = objective(a32.astype(np.float64), y, ref["x"])
    assert abs(p32 - p64) <= 1e-4 * max(abs(p64), 1e-12), (p32, p64)
    # screening stayed safe: every screened coordinate is at 0 in the fp64 optimum
    xs = ref["x"]
    assert np.all(np.abs(xs[res.sat_lower]) <= 1e-6 * max(1.0, np.abs(xs).max()))


def test_fp32_tall_row_blocked():
    """fp32 rows beyond the register-resident envelope (m > 24,576): the
    row-blocked schedule; objective per round tracks the fp64 oracle on the
    same rounded matrix to 1e-4 relative."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(4, m=25000, n=300)
    a64 = np.asfortranarray(inst.a.astype(np.float64))
    g = solve(Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=np.float32),
              SolverConfig(kind="pg", inner_passes=10, gap_tol=1e-9, max_rounds=25))
    o = oracle_solve(a64, inst.y, inst.lower, inst.upper, kind="pg", inner_passes=10, gap_tol=1e-300, max_rounds=25)
    for tg, to in zip(g.trace, o["trace"]):
        assert abs(tg.primal - to["primal"]) <= 1e-4 * abs(to["primal"]), (tg.round, tg.primal, to["primal"])


@pytest.mark.parametrize("family", ["bvls", "mixed"])
@pytest.mark.parametrize("m,n", [(1, 6), (5, 3), (33, 120)])
@pytest.mark.parametrize("kind", ["pg", "apg", "cd"])
def test_bounded_families_edge_shapes(family, m, n, kind):
    from conftest import small_instance
    rng = np.random.default_rng(m * 7 + n)
    a, y, lo, hi = small_instance(rng, m, n, family)
    g, o = _solve_both(a, y, lo, hi, kind, passes=10 if kind != "cd" else 1, tol=1e-9, max_rounds=20)
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]


def test_sharded_more_ranks_than_columns():
    """Column blocks need a column per rank: 3 columns over 4 ranks is refused
    up front (on every rank alike), 4 over 4 runs and matches the oracle."""
    from paper_2202_07258_b200 import Problem, SolverConfig
    from paper_2202_07258_b200.distributed import solve_group
    cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-9, max_rounds=60)
    a, y, lo, hi = _nnls(20, 3, seed=5)
    with pytest.raises(ValueError):
        solve_group(Problem(a, y, lo, hi), cfg, nranks=4)
    a, y, lo, hi = _nnls(20, 4, seed=5)
    g = solve_group(Problem(a, y, lo, hi), cfg, nranks=4)
    o = oracle_solve(a, y, lo, hi, kind="apg", inner_passes=10, gap_tol=1e-9, max_rounds=60)
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]


def test_batched_rejects_tall_dictionary():
    """The batched kernel keeps m <= 208 rows of R in registers: taller
    dictionaries are refused with a clean error, not run wrong."""
    from paper_2202_07258_b200.batched import solve_batched
    rng = np.random.default_rng(1)
    a = np.abs(rng.standard_normal((300, 50)))
    with pytest.raises(Exception):
        solve_batched(a, np.abs(rng.standard_normal((300, 64))), passes=10, rounds=1)


@pytest.mark.parametrize("family", ["nnls", "bvls", "mixed"])
@pytest.mark.parametrize("kind", ["pg", "apg", "cd"])
def test_wide_shapes_reach_the_oracle_optimum(family, kind):
    """m = 2 rows, 5,000 columns: the fit becomes exact within a few rounds,
    after which the residual -- and with it the dual point -- is pure
    round-off, so round-by-round parity at 1e-10 is not a meaningful target
    (hard part 1).  Each solver's objective is within its
    final (certified or reduced) gap of the optimum, so the two objectives
    must agree to the sum of the two gaps; the GPU iterate is feasible."""
    from conftest import small_instance
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    rng = np.random.default_rng(5000 + len(family))
    if family == "nnls":
        a, y, lo, hi = _nnls(2, 5000, seed=3)
    else:
        a, y, lo, hi = small_instance(rng, 2, 5000, family)
    g = solve(Problem(a, y, lo, hi), SolverConfig(kind=kind, inner_passes=10 if kind != "cd" else 1, gap_tol=1e-9,
                                                  max_rounds=1500))
    o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=10 if kind != "cd" else 1, gap_tol=1e-9, max_rounds=1500)
    pg_, po = objective(a, y, np.asarray(g.x)), objective(a, y, o["x"])
    assert abs(pg_ - po) <= g.gap + o["gap"] + 1e-9 * max(1.0, abs(po)), (pg_, po, g.gap, o["gap"])
    assert g.gap <= 1e-3 * max(1.0, abs(po))  # and it got somewhere
    assert np.all(g.x >= lo - 1e-15) and np.all(g.x <= hi + 1e-15)


@pytest.mark.parametrize("family", ["nnls", "bvls", "mixed"])
@pytest.mark.parametrize("m,n", [(40, 7), (9, 9), (200, 3), (1, 1)])
def test_active_set_edge_shapes(family, m, n):
    from conftest import small_instance
    rng = np.random.default_rng(m * 13 + n)
    a, y, lo, hi = small_instance(rng, m, n, family)
    g, o = _solve_both(a, y, lo, hi, "active-set", passes=1, tol=1e-10, max_rounds=None)
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]


@pytest.mark.parametrize("layout", ["row-major", "column-major", "fp32-host"])
def test_device_and_host_inputs_give_the_same_solve(layout):
    """Problem accepts host arrays or CUDA tensors in either layout; the
    device copy has the C-ABI column-major layout either way, so the solves
    are identical (bit for bit) to the numpy-input solve."""
    import torch
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    a, y, lo, hi = _nnls(300, 500, seed=77)
    cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-8, max_rounds=300)
    ref = solve(Problem(a, y, lo, hi), cfg)
    if layout == "row-major":
        p = Problem(torch.from_numpy(np.ascontiguousarray(a)).cuda(), torch.from_numpy(y).cuda(), lo, hi)
    elif layout == "column-major":
        p = Problem(torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t(), torch.from_numpy(y).cuda(), lo, hi)
    else:
        p = Problem(a.astype(np.float32).astype(np.float64), y.astype(np.float32), lo, hi)
    res = solve(p, cfg)
    if layout == "fp32-host":
        a2 = a.astype(np.float32).astype(np.float64)
        y2 = y.astype(np.float32).astype(np.float64)
        ref = solve(Problem(a2, y2, lo, hi), cfg)
    assert res.rounds == ref.rounds
    np.testing.assert_array_equal(np.asarray(res.x), np.asarray(ref.x))
    assert [t.gap for t in res.trace] == [t.gap for t in ref.trace]


def _saturating_bvls(m, n):
    rng = np.random.default_rng(m + n)
    a = np.asfortranarray(rng.standard_normal((m, n)) / np.sqrt(m))
    # 70% of the planted coordinates lie outside the box [-1, 1]
    xt = np.where(rng.random(n) < 0.7, 2.0 * np.sign(rng.standard_normal(n)), rng.uniform(-0.5, 0.5, n))
    y = a @ xt + 0.01 * rng.standard_normal(m)
    return a, y, np.full(n, -1.0), np.full(n, 1.0)


@pytest.mark.parametrize("m,n", [(400, 1200), (3000, 700)])
@pytest.mark.parametrize("kind", ["pg", "apg"])
@pytest.mark.parametrize("streamed", [False, True])
def test_first_order_bvls_screening_both_bounds(m, n, kind, streamed, monkeypatch):
    """Upper- and lower-bound screening (z update with nonzero bounds) on
    both PG / FISTA paths."""
    if streamed:
        monkeypatch.setenv("BX_NO_SMALL", "1")
    else:
        monkeypatch.delenv("BX_NO_SMALL", raising=False)
    a, y, lo, hi = _saturating_bvls(m, n)
    g, o = _solve_both(a, y, lo, hi, kind, passes=10, tol=1e-9, max_rounds=200)
    assert len(o["sat_lower"]) > 0 and len(o["sat_upper"]) > 0
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]


@pytest.mark.parametrize("m,n", [(400, 1200), (3000, 700)])
def test_cd_with_screening_events(m, n):
    """Coordinate descent on a box-constrained family whose optimum saturates
    many coordinates: screening fires while the sweep spans many blocks, so
    compaction, the Gram / cross-Gram recompute and the pipelined block ring
    all run between sweeps (m = 3000 also takes the two-slot ring)."""
    a, y, lo, hi = _saturating_bvls(m, n)
    g, o = _solve_both(a, y, lo, hi, "cd", passes=1, tol=1e-9, max_rounds=150)
    assert o["trace"][-1]["preserved"] < n  # screening fired
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]


@pytest.mark.parametrize("m,n,K", [(1, 5, 1), (8, 15, 63), (37, 17, 65), (208, 40, 64), (50, 33, 129)])
@pytest.mark.parametrize("screening", [True, False])
def test_batched_edge_shapes(m, n, K, screening):
    """Batched many-RHS FISTA: a partial last problem tile (K % 64), a
    dictionary narrower than one 16-column chunk or with a ragged last chunk,
    a single row, the 208-row register envelope; per problem vs the batched
    oracle."""
    from oracle.batched_oracle import batched_apg
    from paper_2202_07258_b200.batched import solve_batched
    rng = np.random.default_rng(m * 1000 + n * 10 + K)
    a = np.abs(rng.standard_normal((m, n))) + 0.05
    X0 = np.zeros((n, K))
    for k in range(K):
        sup = rng.choice(n, size=min(3, n), replace=False)
        X0[sup, k] = rng.random(sup.size)
    Y = a @ X0 + 0.05 * rng.standard_normal((m, K))
    g = solve_batched(a, Y, passes=10, rounds=6, gap_tol=1e-300, screening=screening)
    o = batched_apg(a, Y, eta=g.eta, inner_passes=10, rounds=6, gap_tol=1e-300, screening=screening)
    # both stop early when every gap reaches exactly 0 (m = 1: exact fit)
    assert g.rounds == len(o["gap"])
    scale = np.maximum(np.maximum(np.abs(o["primal"][-1]), np.abs(o["dual"][-1])), 1e-3)
    for name, gv in (("primal", g.primal), ("dual", g.dual), ("gap", g.gap)):
        d = np.abs(gv - o[name][-1])
        assert np.all(d <= 1e-10 * scale), (name, d.max())
    np.testing.assert_array_equal(g.preserved, o["preserved"][-1])
    assert np.max(np.abs(g.x - o["X"])) <= 1e-8 * max(1.0, np.abs(o["X"]).max())


def test_batched_stops_when_every_problem_converged():
    from paper_2202_07258_b200.batched import solve_batched
    rng = np.random.default_rng(3)
    a = np.abs(rng.standard_normal((60, 20))) + 0.1
    Y = a @ np.abs(rng.standard_normal((20, 64)))
    g = solve_batched(a, Y, passes=10, rounds=200, gap_tol=1e-3)
    assert g.converged == 64 and g.rounds < 200 and np.all(g.gap < 1e-3)

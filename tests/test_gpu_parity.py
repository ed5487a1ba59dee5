"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, round by round."""

import zlib

import numpy as np
import pytest

from conftest import small_instance
from oracle.boxscreen_oracle import oracle_solve
from parity import compare_final, compare_traces

pytestmark = pytest.mark.gpu


def _solve_both(a, y, lo, hi, kind, passes=10, tol=1e-8, screening=True, max_rounds=None):
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    p = Problem(a, y, lo, hi)
    g = solve(p, SolverConfig(kind=kind, inner_passes=passes, gap_tol=tol, max_rounds=max_rounds),
              screening=screening)
    o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=passes, gap_tol=tol, screening=screening,
                     max_rounds=max_rounds)
    return g, o


@pytest.fixture(params=["resident", "streamed"])
def path(request, monkeypatch):
    """Run PG / FISTA rounds on the cooperative SM-resident kernel (small
    problems, bx_small.cuh) or force the streamed k_pass + k_reduce path."""
    if request.param == "streamed":
        monkeypatch.setenv("BX_NO_SMALL", "1")
    else:
        monkeypatch.delenv("BX_NO_SMALL", raising=False)
    return request.param


@pytest.mark.parametrize("family", ["nnls", "bvls", "mixed"])
@pytest.mark.parametrize("kind", ["pg", "apg", "cd"])
@pytest.mark.parametrize("screening", [True, False])
def test_small_trajectories(family, kind, screening, path):
    rng = np.random.default_rng(zlib.crc32(f"{family}-{kind}-{screening}".encode()))
    for _ in range(4):
        n = int(rng.integers(3, 31))
        m = int(rng.integers(n, 61))
        a, y, lo, hi = small_instance(rng, m, n, family)
        g, o = _solve_both(a, y, lo, hi, kind, screening=screening)
        probs = compare_traces(g, o) + compare_final(g, o)
        assert not probs, (family, kind, m, n, probs[:3])


def test_kat_1d_nnls_converges_in_one_round():
    # test_driver.py:15-22: A=[[1]], y=[-1], NNLS -> x=0, one round, ratio 1
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    res = solve(Problem([[1.0]], [-1.0], 0.0, np.inf), SolverConfig(kind="pg"), screening=True)
    assert res.converged and res.rounds == 1
    assert res.x[0] == 0.0 and res.gap < 1e-12
    assert res.trace[-1].screening_ratio == 1.0


def test_pg_explicit_step_kat():
    # test_solvers.py:78-83: A=[[1]], y=[3], box [0,1], step 1 -> x = 1
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    res = solve(Problem([[1.0]], [3.0], 0.0, 1.0), SolverConfig(kind="pg", step_size=1.0, max_rounds=1),
                screening=False)
    assert res.x[0] == 1.0


def test_step_too_large_raises():
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.errors import StepSizeTooLarge
    rng = np.random.default_rng(3)
    a = rng.standard_normal((10, 6))
    sigma = np.linalg.svd(a, compute_uv=False)[0]
    p = Problem(a, rng.standard_normal(10) * 5, -10.0, 10.0)
    with pytest.raises(StepSizeTooLarge):
        solve(p, SolverConfig(kind="pg", step_size=2.5 / sigma ** 2, max_rounds=50, inner_passes=1),
              screening=False)


def test_zero_column_and_interior():
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.errors import NoInteriorPoint, ZeroColumn
    a = np.array([[1.0, 0.0], [1.0, 0.0]])
    with pytest.raises(NoInteriorPoint):
        solve(Problem(a, np.zeros(2), 0.0, np.inf), SolverConfig(kind="pg"))
    with pytest.raises(ZeroColumn):
        solve(Problem(a, np.zeros(2), 0.0, 1.0), SolverConfig(kind="pg"))


@pytest.mark.parametrize("cfg_id,m,n,rounds", [(1, 1000, 2000, 300), (3, 1000, 5000, 200), (2, 500, 1000, 60)])
def test_baseline_recipe_prefix(cfg_id, m, n, rounds, path):
    """BASELINE config recipes at oracle-friendly sizes: first rounds round-by-round."""
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(cfg_id, m=m, n=n)
    g, o = _solve_both(inst.a, inst.y, inst.lower, inst.upper, inst.kind, passes=inst.inner_passes,
                       tol=inst.gap_tol, max_rounds=rounds)
    probs = compare_traces(g, o)
    assert not probs, probs[:3]


@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_tall_matrix_row_blocked_path(kind):
    """m = 13000 fp64 rows is beyond the register-resident fused pass: the
    row-blocked path (dot over row blocks, column update, A x blocks) must
    follow the oracle round by round."""
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(3, m=13000, n=600)
    g, o = _solve_both(inst.a, inst.y, inst.lower, inst.upper, kind, passes=10, tol=1e-6, max_rounds=40)
    probs = compare_traces(g, o)
    assert not probs, probs[:3]


@pytest.mark.parametrize("m,n", [(4500, 300), (2000, 70), (2000, 40)])
def test_cd_block_pipeline_shapes(m, n):
    """Coordinate descent shapes off the config-2 path: m = 4500 leaves room
    for only two shared-memory block slots (the next block's copy waits for
    the axpy), and n = 70 / 40 give passes of three / two blocks, where the
    column-state look-ahead takes x from the redundant update instead of
    global memory; 10 sweeps per round exercise the cross-pass hand-off."""
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(2, m=m, n=n)
    g, o = _solve_both(inst.a, inst.y, inst.lower, inst.upper, "cd", passes=10, tol=1e-9, max_rounds=15)
    probs = compare_traces(g, o) + compare_final(g, o)
    assert not probs, probs[:3]

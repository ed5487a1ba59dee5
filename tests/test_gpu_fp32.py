"""fp32 storage of A + fp32 accumulation of the streamed products (BASELINE
config 4) against the fp64 oracle on the same (fp32-rounded) matrix: objective
within 1e-4 relative (north_star), screened coordinates saturated in a
high-accuracy fp64 solution (safety).  The fp32 stop rule is the relative gap
gap <= gap_tol * max(1, P) ("fp32")."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_fp32_config4_recipe(kind):
    from oracle.boxscreen_oracle import objective, oracle_solve
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(4, m=1500, n=4000)            # fp32 A, fp64 y
    assert inst.a.dtype == np.float32
    a64 = np.asfortranarray(inst.a.astype(np.float64))  # the same (rounded) matrix in fp64
    res = solve(Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=np.float32),
                SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-6 if kind == "apg" else 1e-5,
                             max_rounds=40000))
    assert res.converged, (res.rounds, res.gap, res.trace[-1].primal)
    ref = oracle_solve(a64, inst.y, inst.lower, inst.upper, kind="apg", inner_passes=10, gap_tol=1e-9)
    assert ref["converged"]
    p32 = objective(a64, inst.y, np.asarray(res.x, dtype=np.float64))
    p64 = objective(a64, inst.y, ref["x"])
    assert abs(p32 - p64) <= 1e-4 * abs(p64), (p32, p64)
    # every coordinate the fp32 run screened is at its bound in the fp64 optimum
    xs = ref["x"]
    assert np.all(np.abs(xs[res.sat_lower]) <= 1e-6 * max(1.0, np.abs(xs).max()))
    assert res.sat_lower.size > 0


def test_fp32_matches_fp64_trajectory_early():
    """Early rounds of fp32 PG track the fp64 oracle to fp32 resolution."""
    from oracle.boxscreen_oracle import oracle_solve
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(4, m=1000, n=2000)
    a64 = np.asfortranarray(inst.a.astype(np.float64))
    res = solve(Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=np.float32),
                SolverConfig(kind="pg", inner_passes=10, gap_tol=1e-6, max_rounds=50))
    o = oracle_solve(a64, inst.y, inst.lower, inst.upper, kind="pg", inner_passes=10, gap_tol=1e-6, max_rounds=50)
    for g, r in zip(res.trace, o["trace"]):
        assert abs(g.primal - r["primal"]) <= 1e-4 * abs(r["primal"])

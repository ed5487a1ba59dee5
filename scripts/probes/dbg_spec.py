import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_gpu_edges import _saturating_bvls
from oracle.boxscreen_oracle import oracle_solve
from paper_2202_07258_b200 import Problem, SolverConfig, solve
a, y, lo, hi = _saturating_bvls(400, 1200)
o = oracle_solve(a, y, lo, hi, kind="pg", inner_passes=10, gap_tol=1e-9, max_rounds=200)
print("oracle rounds", o["rounds"], "conv", o["converged"])
g = solve(Problem(a, y, lo, hi), SolverConfig(kind="pg", inner_passes=10, gap_tol=1e-9, max_rounds=200))
d = np.abs(g.x - o["x"]); bad = np.flatnonzero(d > 1e-8)
print(os.environ.get("TAG"), "rounds", g.rounds, "maxdiff", d.max(), "nbad", bad.size, "info", {k: g.info[k] for k in ("spec_kept", "spec_undone", "iterations")})
print(" bad idx", bad[:10], "gpu", g.x[bad[:5]], "orc", o["x"][bad[:5]])
print(" in sat_lo", np.isin(bad, g.sat_lower).sum(), "in sat_up", np.isin(bad, g.sat_upper).sum())
print(" trace last", g.trace[-1].primal, o["trace"][-1]["primal"])
from oracle.boxscreen_oracle import objective
print(" obj(gpu x)", objective(a, y, g.x), "obj(orc x)", objective(a, y, o["x"]))

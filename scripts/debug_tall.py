import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2202_07258_b200 import Problem, SolverConfig, solve, spectral_norm_estimate
from paper_2202_07258_b200.generate import make_config
from oracle.boxscreen_oracle import oracle_solve, spectral_sigma
inst = make_config(3, m=13000, n=600)
print("sigma gpu", spectral_norm_estimate(inst.a), "oracle", spectral_sigma(inst.a))
for passes in (1, 2):
    for kind in ("pg", "apg"):
        p = Problem(inst.a, inst.y, inst.lower, inst.upper)
        g = solve(p, SolverConfig(kind=kind, inner_passes=passes, gap_tol=1e-6, max_rounds=1), screening=False)
        o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind=kind, inner_passes=passes, gap_tol=1e-6, max_rounds=1, screening=False)
        print(kind, passes, "P", g.trace[0].primal, o["trace"][0]["primal"], "D", g.trace[0].dual, o["trace"][0]["dual"], "step", g.info["step"], o["step"], "dx", np.abs(g.x - o["x"]).max())

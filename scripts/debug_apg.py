"""Debug helper: find APG instances whose GPU trajectory departs from the oracle
and locate the first differing round (x vectors compared round by round)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import small_instance
from oracle.boxscreen_oracle import oracle_solve
from parity import compare_traces
from paper_2202_07258_b200 import Problem, SolverConfig, solve

fam = sys.argv[1] if len(sys.argv) > 1 else "nnls"
kind = sys.argv[2] if len(sys.argv) > 2 else "apg"
nfail = 0
for seed in range(40):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 31)); m = int(rng.integers(n, 61))
    a, y, lo, hi = small_instance(rng, m, n, fam)
    p = Problem(a, y, lo, hi)
    g = solve(p, SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-8))
    restarts = []
    o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=10, gap_tol=1e-8)
    probs = compare_traces(g, o)
    if not probs:
        continue
    nfail += 1
    print("seed", seed, m, n, probs[0])
    # locate first round where x differs
    for r in range(1, len(o["trace"]) + 1):
        gr = solve(p, SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-8, max_rounds=r))
        orr = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=10, gap_tol=1e-8, max_rounds=r)
        dx = np.max(np.abs(gr.x - orr["x"]))
        print("  round", r, "max|dx|=%.3e" % dx, "P gpu-orc=%.3e" % (gr.trace[-1].primal - orr["trace"][-1]["primal"]),
              "preserved", gr.trace[-1].preserved_count, orr["trace"][-1]["preserved"], "step", gr.info["step"], orr["step"])
        if dx > 1e-9:
            break
    if nfail >= 2:
        break
print("failures", nfail)

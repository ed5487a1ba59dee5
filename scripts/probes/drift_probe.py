"""Per-round deviation of the GPU trajectory from the oracle (P, D relative to
max(|P|, |D|)) for the instance of test_rounds_through_fine_grained_abi."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from conftest import small_instance
from oracle.boxscreen_oracle import oracle_solve
from paper_2202_07258_b200 import Problem, SolverConfig, solve
for fam in ("nnls", "mixed"):
    rng = np.random.default_rng(77 + ["nnls", "bvls", "mixed"].index(fam))
    a, y, lo, hi = small_instance(rng, 120, 300, fam)
    for kind in ("apg", "pg"):
        o = oracle_solve(a, y, lo, hi, kind=kind, inner_passes=10, gap_tol=1e-9, max_rounds=80)
        for env in ("", "BX_SPEC=0", "BX_NO_SMALL=1"):
            for k in ("BX_SPEC", "BX_NO_SMALL"):
                os.environ.pop(k, None)
            if env:
                kk, vv = env.split("="); os.environ[kk] = vv
            g = solve(Problem(a, y, lo, hi), SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-9, max_rounds=80))
            dev = []
            for gt, ot in zip(g.trace, o["trace"]):
                sc = max(abs(ot["primal"]), abs(ot["dual"]))
                dev.append(max(abs(gt.primal - ot["primal"]), abs(gt.dual - ot["dual"])) / sc)
            dev = np.array(dev)
            print(fam, kind, env or "default", "rounds", len(g.trace), len(o["trace"]), "max rel dev %.2e at %d" % (dev.max(), dev.argmax() + 1),
                  "dev@10/30/50: %s" % ", ".join("%.1e" % dev[i] for i in (9, 29, 49) if i < dev.size), flush=True)

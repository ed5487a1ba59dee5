"""Time config 3's first 40 rounds (fused reduce debug stamps via BX_DBG_FUSE)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2202_07258_b200 import Problem, SolverConfig, solve
from paper_2202_07258_b200.generate import make_config
inst = make_config(3)
p = Problem(inst.a, inst.y, inst.lower, inst.upper)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    r = solve(p, SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=40))
    torch.cuda.synchronize(); print("40 rounds %.3f s" % (time.time() - t0), flush=True)

"""ncu target: one round of the batched DMMA kernel over 148 tiles (9472 RHS) of config 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2202_07258_b200.batched import solve_batched
from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
a = bump_dictionary(200, 5000)
Y, _ = batched_rhs(a, 148 * 64)
r = solve_batched(a, Y, passes=10, rounds=1, gap_tol=1e-6, return_device=True)
torch.cuda.synchronize()
print("rounds", r.rounds, "mean gap", r.gap.mean())

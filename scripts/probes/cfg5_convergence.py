"""Config 5 (K = 100,000 RHS): rounds to the per-problem gap and screening
over the solve (max gap, mean preserved, time per round)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2202_07258_b200.batched import solve_batched
from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
from paper_2202_07258_b200.solvers import auto_step_size
a = bump_dictionary(200, 5000)
Y, _ = batched_rhs(a, 100000)
eta = auto_step_size(a, 1.0)
ad = torch.from_numpy(a).cuda(); yd = torch.from_numpy(np.ascontiguousarray(Y)).cuda()
for rounds in (2, 20, 100, 400, 1600):
    torch.cuda.synchronize(); t0 = time.time()
    r = solve_batched(ad, yd, passes=10, rounds=rounds, gap_tol=1e-6, eta=eta, return_device=True)
    torch.cuda.synchronize(); dt = time.time() - t0
    g = r.gap.cpu().numpy() if hasattr(r.gap, "cpu") else np.asarray(r.gap)
    pres = r.preserved.cpu().numpy() if hasattr(r.preserved, "cpu") else np.asarray(r.preserved)
    print(f"rounds {rounds:5d} ran {r.rounds:5d} {dt:8.2f}s  max_gap {g.max():.3e} median_gap {np.median(g):.3e} "
          f"frac<1e-6 {np.mean(g < 1e-6):.4f} mean_preserved {pres.mean():.1f} min {pres.min()}", flush=True)

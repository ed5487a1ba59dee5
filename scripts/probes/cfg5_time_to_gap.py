"""Config 5 (K = 100,000 RHS): one long batched solve (16 rounds per launch),
time to looser per-problem gap levels from the per-round trace (the stated
1e-6 is out of reach on the correlated bump dictionary).
usage: cfg5_time_to_gap.py [rounds]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2202_07258_b200.batched import solve_batched
from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
from paper_2202_07258_b200.solvers import auto_step_size
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
a = bump_dictionary(200, 5000)
Y, _ = batched_rhs(a, 100000)
eta = auto_step_size(a, 1.0)
ad = torch.from_numpy(a).cuda(); yd = torch.from_numpy(np.ascontiguousarray(Y)).cuda()
solve_batched(ad, yd, passes=10, rounds=2, gap_tol=1e-6, eta=eta, return_device=True)
torch.cuda.synchronize(); t0 = time.time()
r = solve_batched(ad, yd, passes=10, rounds=rounds, gap_tol=1e-6, eta=eta, return_device=True, check_every=16)
torch.cuda.synchronize(); dt = time.time() - t0
per = dt / r.rounds
print(f"{r.rounds} rounds ({r.iterations} FISTA steps on each of 100,000 right-hand sides) in {dt:.1f} s "
      f"= {per * 1e3:.1f} ms per round, {r.iterations * 100000 / dt / 1e6:.2f} M rhs-iterations/s; "
      f"sphere sweeps run: {r.sphere_sweeps} of {r.rounds * r.tiles} tile-rounds")
tr = r.trace  # converged, max gap, mean gap, mean preserved
for level in (1e-1, 1e-2, 1e-3, 1e-4, 3e-5):
    hit = np.nonzero(tr[:, 1] <= level)[0]
    print(f"max gap over all problems <= {level:.0e}: " + (f"round {hit[0] + 1}, {per * (hit[0] + 1):7.1f} s" if hit.size else "not reached"))
for level in (1e-3, 1e-4, 1e-5):
    hit = np.nonzero(tr[:, 2] <= level)[0]
    print(f"mean gap <= {level:.0e}: " + (f"round {hit[0] + 1}, {per * (hit[0] + 1):7.1f} s" if hit.size else "not reached"))
g = np.asarray(r.gap)
print(f"final: max gap {g.max():.3e}, median {np.median(g):.3e}, below 1e-6: {np.mean(g < 1e-6):.4f}, mean preserved {r.preserved.mean():.1f}")

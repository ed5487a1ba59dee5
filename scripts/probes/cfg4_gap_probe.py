"""Config 4's single-GPU shard (20000 x 62,500 fp32, PG, screening): rounds and
time to a relative certified gap (gap <= tol * max(1, P)) for a few tols."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench
from paper_2202_07258_b200 import Problem, SolverConfig, solve
inst = bench.make_instance(4)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
for kind in ("pg", "apg"):
    for tol in (1e-3, 1e-4, 1e-5):
        torch.cuda.synchronize(); t0 = time.time()
        r = solve(p, SolverConfig(kind=kind, inner_passes=10, gap_tol=tol, max_rounds=20000, relative_gap=True),
                  return_device=True)
        torch.cuda.synchronize(); dt = time.time() - t0
        print(f"{kind} rel tol {tol:g}: converged {r.converged} rounds {r.rounds} iters {r.info['iterations']} "
              f"{dt:.2f}s preserved {r.trace[-1].preserved_count} gap {r.gap:.3e} P {r.trace[-1].primal:.6e}", flush=True)

"""Config 4 weak-scaling unit (20000 x 62500 fp32): iteration rate and gap
progress of a capped PG solve (how long a full solve to gap takes)."""
import sys
import time

import numpy as np
import torch

sys.argv = ["bench"]
import bench  # noqa: E402
from paper_2202_07258_b200 import Problem, SolverConfig, solve  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 300
inst = bench.make_instance(4)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
for kind, passes in (("pg", 10), ("apg", 10)):
    cfg = SolverConfig(kind=kind, inner_passes=passes, gap_tol=1e-6, max_rounds=cap)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = solve(p, cfg, return_device=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    tr = r.info["trace_arrays"]
    print(f"{kind}: {r.rounds} rounds in {el:.2f}s ({r.info['iterations'] / el:.0f} it/s) conv={r.converged}")
    for i in list(range(0, len(tr), max(1, len(tr) // 12))) + [len(tr) - 1]:
        rec = tr[i]
        print(f"  round {rec['round']:6d} P={rec['primal']:.6e} gap={rec['gap']:.3e} rel={rec['gap'] / max(1, rec['primal']):.3e} k={rec['preserved_count']}")

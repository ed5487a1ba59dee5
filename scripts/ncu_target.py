"""Short, ncu-friendly run of the hot path: BASELINE config 3 at full size
(10000 x 50000 fp64), FISTA with screening, first 3 rounds only (33 fused
passes + 3 screening passes).  Used for the ncu launch list and the full
capture of the fused pass kernel (profiles/)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2202_07258_b200 import Problem, SolverConfig, solve
from paper_2202_07258_b200.generate import make_config
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
inst = make_config(cfg_id)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
res = solve(p, SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol, max_rounds=rounds),
            return_device=True)
torch.cuda.synchronize()
print("rounds", res.rounds, "launches", res.info["kernel_launches"])

"""Short, ncu-friendly run of the hot path of one BASELINE config (its
single-GPU workload, bench.make_instance), first few rounds only.  Used for
the ncu launch lists and the full captures summarised under profiles/.

    python scripts/ncu_target.py CONFIG [ROUNDS] [KIND]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = sys.argv[3] if len(sys.argv) > 3 else None
argv, sys.argv = sys.argv, sys.argv[:1]
import bench  # noqa: E402
from paper_2202_07258_b200 import Problem, SolverConfig, solve  # noqa: E402

inst = bench.make_instance(cfg_id)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
res = solve(p, SolverConfig(kind=kind or inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol,
                            max_rounds=rounds), return_device=True)
torch.cuda.synchronize()
print("rounds", res.rounds, "launches", res.info["kernel_launches"])

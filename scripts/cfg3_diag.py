"""GPU diagnostics for the config-3 trajectory: restarts, momentum and gap per round."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2202_07258_b200 import Problem, SolverConfig, solve
from paper_2202_07258_b200.generate import make_config
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = make_config(cfg_id)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
res = solve(p, SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol), return_device=True)
tr = res.info["trace_arrays"]
print("rounds", res.rounds, "iters", res.info["iterations"], "restarts", res.info["restarts"], "conv", res.converged)
idx = np.unique(np.r_[np.arange(0, len(tr), max(1, len(tr)//40)), len(tr)-1])
for i in idx:
    r = tr[i]
    print(int(r["round"]), "P=%.10e gap=%.3e k=%d eps=%.3e step=%.3e restarts=%d t=%.1f" % (r["primal"], r["gap"], r["preserved_count"], r["eps"], r["step"], r["restarts"], r["momentum"]))
np.save("gpurun_out/cfg%d_trace.npy" % cfg_id, tr)

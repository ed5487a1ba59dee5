"""Time the active-set kind on BASELINE config 1's instance (GPU)."""
import time

import numpy as np
import torch

from paper_2202_07258_b200 import Problem, SolverConfig, solve
from paper_2202_07258_b200.generate import make_config

inst = make_config(1)
p = Problem(inst.a, inst.y, inst.lower, inst.upper)
cfg = SolverConfig(kind="active-set", gap_tol=1e-6)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = solve(p, cfg)
    torch.cuda.synchronize()
    print(f"rep {rep}: {time.perf_counter() - t:.3f} s rounds={r.rounds} conv={r.converged} "
          f"launches={r.info['kernel_launches']} gap={r.gap:.3e}")
r = solve(p, cfg, profile=True)
for k, v in sorted(r.info["profile"].items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:12s} launches={v['launches']:7d} ms={v['ms']:9.3f}")

"""Sustained-load timing of the fused FISTA pass (config 3, first 60 rounds,
k = n): per-launch time of pass_apg for back-to-back solves, with the SM clock
and throttle reasons sampled by nvidia-smi, to separate clock / power effects
from the kernel itself."""
import subprocess
import sys
import time

import numpy as np
import torch

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2202_07258_b200 import Problem, SolverConfig, solve  # noqa: E402


def smi():
    q = "clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"], capture_output=True,
                          text=True).stdout.strip()


inst = bench.make_instance(3)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
cfg = SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol, max_rounds=60)
for it in range(N):
    t = time.perf_counter()
    rp = solve(p, cfg, return_device=True, profile=True)
    torch.cuda.synchronize()
    e = rp.info["profile"]["pass_apg"]
    d = rp.info["profile"]["pass_dot"]
    print(f"solve {it}: wall {time.perf_counter() - t:.2f}s k={rp.trace[-1].preserved_count} "
          f"pass_apg {e['ms'] / e['launches'] * 1e3:.1f} us/launch {e['bytes'] / (e['ms'] / 1e3) / 1e9:.0f} GB/s | "
          f"pass_dot {d['bytes'] / (d['ms'] / 1e3) / 1e9:.0f} GB/s | smi {smi()}", flush=True)

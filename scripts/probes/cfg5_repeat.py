"""Config 5: time per solve_batched call (2 rounds) repeated in one process;
run several processes to separate per-process (memory placement) from
per-call variation.  usage: cfg5_repeat.py [K] [calls] [rounds] [check_every]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2202_07258_b200.batched import solve_batched
from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
from paper_2202_07258_b200.solvers import auto_step_size
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
every = int(sys.argv[4]) if len(sys.argv) > 4 else 1
a = bump_dictionary(200, 5000)
Y, _ = batched_rhs(a, K)
dev = torch.device("cuda")
a_dev = torch.from_numpy(a).to(dev)
y_dev = torch.from_numpy(np.ascontiguousarray(Y)).to(dev)
eta = auto_step_size(a, 1.0)
ts = []
for i in range(calls):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = solve_batched(a_dev, y_dev, passes=10, rounds=rounds, gap_tol=1e-6, eta=eta, return_device=True, check_every=every)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
flops = rounds * 42.0 * 200 * 5000 * K
print(f"rounds {rounds} check_every {every}: rhs-it/s {10 * rounds * K / (min(ts) / 1e3) / 1e6:.3f} M;", "ms per call:", " ".join(f"{t:.1f}" for t in ts), "| TFLOP/s best %.2f last %.2f" % (flops / min(ts) / 1e9, flops / ts[-1] / 1e9))

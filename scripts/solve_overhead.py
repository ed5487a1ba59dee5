"""Host-side overhead of one solve() call: session creation, native loop,
result conversion (config 3 capped at a few rounds)."""
import sys
import time

import numpy as np
import torch

sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2202_07258_b200 import Problem, SolverConfig, driver  # noqa: E402

inst = bench.make_instance(3)
a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=20)
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = driver._Session(p)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out, tr, x, theta, sl, su = s.run(cfg, True, 1.0, 1e-12)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = driver._result(p.n, out, tr, x, theta, sl, su, None, True)
    s.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {rep}: session {1e3 * (t1 - t0):.1f} ms  run {1e3 * (t2 - t1):.1f} ms  result+close {1e3 * (t3 - t2):.1f} ms"
          f"  launches {out.kernel_launches}")

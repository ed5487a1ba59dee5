"""A/B timing of the streamed pass: configs 3 and 4, a fixed number of
rounds, per-kernel live profile (GB/s of the fused pass) and wall time."""
import sys
import time

import numpy as np
import torch

sys.argv = sys.argv[:1]
import bench  # noqa: E402
from paper_2202_07258_b200 import Problem, SolverConfig, solve  # noqa: E402

for cfg_id, rounds in ((3, 60), (4, 40)):
    inst = bench.make_instance(cfg_id)
    a_dev = torch.from_numpy(np.ascontiguousarray(inst.a.T)).cuda()
    p = Problem(a_dev.t(), torch.from_numpy(inst.y).cuda(), inst.lower, inst.upper)
    cfg = SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol, max_rounds=rounds)
    solve(p, cfg, return_device=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = solve(p, cfg, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    rp = solve(p, cfg, return_device=True, profile=True)
    pr = rp.info["profile"]
    key = "pass_apg" if inst.kind == "apg" else "pass_pg"
    e = pr[key]
    ktot = sum(v["ms"] for v in pr.values())
    print(f"cfg{cfg_id}: {r.info['iterations'] / wall:.1f} it/s wall={wall:.3f}s kernels={ktot / 1e3:.3f}s "
          f"launches={r.info['kernel_launches']} it={r.info['iterations']} k={r.trace[-1].preserved_count} "
          f"{key} {e['bytes'] / (e['ms'] / 1e3) / 1e9:.0f} GB/s ({e['ms'] / e['launches'] * 1e3:.1f} us/launch) "
          + " ".join(f"{k}={v['ms']:.1f}" for k, v in sorted(pr.items(), key=lambda kv: -kv[1]['ms'])[:6]),
          flush=True)
    del p, a_dev
    torch.cuda.empty_cache()

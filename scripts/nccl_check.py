"""Run under torchrun (any number of ranks, one GPU each): an NCCL
column-sharded solve of a reduced config-3 instance must reproduce the
single-context solve (every rank prints its verdict; exit 1 on mismatch)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, torch.distributed as dist
from paper_2202_07258_b200 import Problem, SolverConfig, solve
from paper_2202_07258_b200.distributed import column_blocks, shard, solve_distributed
from paper_2202_07258_b200.generate import make_config
from parity import compare_traces

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
inst = make_config(3, m=800, n=4000)
p = Problem(inst.a, inst.y, inst.lower, inst.upper)
cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=300)
ref = solve(p, cfg)
c0, c1 = column_blocks(p.n, world)[rank]
orc = dict(trace=[dict(primal=t.primal, dual=t.dual, gap=t.gap, preserved=t.preserved_count) for t in ref.trace])
ok = True
# both transports of the per-step reduction: the fused reduce + peer
# exchange kernel (CUDA IPC buffers) and the NCCL allreduce schedule
for exchange in ("fused", "nccl"):
    res = solve_distributed(shard(p, c0, c1), c0, p.n, cfg, return_device=False, exchange=exchange)
    probs = compare_traces(res, orc)
    dx = float(np.max(np.abs(res.x - ref.x[c0:c1]))) if c1 > c0 else 0.0
    good = not probs and dx <= 1e-8 * max(1.0, float(np.max(np.abs(ref.x))))
    ok = ok and good
    print(f"rank {rank}/{world} [{exchange}]: rounds {res.rounds} vs {ref.rounds}, max|dx| {dx:.2e}, "
          f"launches {res.info['kernel_launches']}, {'OK' if good else 'MISMATCH ' + str(probs[:2])}", flush=True)
from paper_2202_07258_b200.distributed import release_comms  # noqa: E402
release_comms()
dist.destroy_process_group()
sys.exit(0 if ok else 1)

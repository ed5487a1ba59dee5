"""Column-sharded solves (BASELINE configs 3 and 4).

Each rank owns a contiguous block of columns (its own A shard, per-column
state and compaction); y, t, z and the residual are replicated.  Per FISTA /
PG step the native loop allreduces the m-vector of partial A x (SUM), per
round the epsilon of the dual translation (MAX), the bound terms of the dual
objective (SUM) and the screening counts (SUM); power iteration and the
certified gap follow the same pattern (csrc/bx_core.cu, run_reduce /
dual_point / global_k).  Two transports behind one C++ interface:

* NCCL (``solve_distributed``): one process per GPU under torchrun; the
  128-byte unique id travels over the caller's torch.distributed group.
* in-process group (``solve_group``): ranks are threads of one process with
  their own streams, synchronised by host barriers only -- the test transport
  that runs the exact sharded code path on a single GPU.

The per-step reduction (the hot collective: once per PG / FISTA step) runs
by default as ONE fused kernel per rank that reduces the pass's partial rows
and exchanges them over peer memory (CUDA IPC mappings, NVLink / NVSwitch),
``csrc/bx_exchange.cuh``; ``exchange="nccl"`` (or BX_EXCHANGE=nccl) keeps it
on NCCL allreduces.  On the in-process group the fused exchange of all ranks
runs as one cooperative launch over their buffers.

Coordinate descent is sequential and is not sharded (replicas only).
"""

import ctypes
import os
import threading

from . import _native as nat
from .driver import _Session, _default_slack, _result
from .model import Problem, QuadraticLoss
from .solvers import SolverConfig


def column_blocks(n, world):
    """Contiguous, balanced column blocks [(c0, c1)] for ``world`` ranks
    (every rank owns at least one column: n >= world)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if n < world:
        raise ValueError(f"{n} columns cannot be sharded over {world} ranks (each rank needs one)")
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def agree_all(ok, pg=None):
    """True iff ``ok`` holds on every rank of ``pg`` (MIN all-reduce; the
    tensor lives where the group's backend wants it)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(pg) == "nccl" else torch.device("cpu")
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=pg)
    return bool(t.item())


def shard(p, c0, c1):
    """Problem over columns [c0, c1) of p, sharing p's device storage."""
    d = p.device_arrays()
    return Problem.from_device_storage(d["a"][c0:c1], p.m, d["y"], d["lo"][c0:c1], d["hi"][c0:c1])


def _exchange(exchange, group=False):
    ex = exchange or os.environ.get("BX_EXCHANGE", "fused")
    allowed = ("fused", "nccl", "peer") if group else ("fused", "nccl")
    if ex not in allowed:
        raise ValueError(f"exchange must be one of {allowed}, not {ex!r}")
    return ex


def solve_group(p, cfg=None, nranks=2, screening=True, tv=None, loss=QuadraticLoss, slack_scale=None,
                return_shards=False, exchange=None):
    """Column-sharded solve with ``nranks`` ranks as threads on the current GPU.

    ``exchange``: "fused" (every rank's reduce + exchange in one cooperative
    launch), "nccl" (the collective schedule through the group's allreduce) or
    "peer" -- each rank thread launches the production exchange kernel
    (``k_xreduce``, what a multi-GPU run launches per GPU) on its own stream;
    the ranks' grids are co-resident and talk through the peer flags."""
    import torch
    cfg = cfg or SolverConfig()
    slack_scale = _default_slack(p) if slack_scale is None else slack_scale
    L = nat.lib()
    group = ctypes.c_void_p()
    ex = _exchange(exchange, group=True)
    prev = os.environ.get("BX_GROUP_XREDUCE")
    os.environ["BX_GROUP_XREDUCE"] = "rank" if ex == "peer" else "group"
    try:
        nat.check(L.bx_group_create(ctypes.byref(group), nranks), None, "bx_group_create")
    finally:
        if prev is None:
            os.environ.pop("BX_GROUP_XREDUCE", None)
        else:
            os.environ["BX_GROUP_XREDUCE"] = prev
    blocks = column_blocks(p.n, nranks)
    sessions, results, errors = [], [None] * nranks, [None] * nranks
    try:
        for r, (c0, c1) in enumerate(blocks):
            s = _Session(shard(p, c0, c1), tv=tv, stream=torch.cuda.Stream())
            s.attach_group(group, r, c0, p.n)
            sessions.append(s)
            if ex in ("fused", "peer"):
                s.attach_peers()

        def work(r):
            try:
                results[r] = sessions[r].run(cfg, screening, loss.alpha, slack_scale)
            except BaseException as e:  # surfaced below
                errors[r] = e

        threads = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errors:
            if e is not None:
                raise e
    finally:
        for s in sessions:
            s.close()
        L.bx_group_destroy(group)
    if return_shards:
        return results
    out, tr, _, theta, _, _ = results[0]
    x = torch.cat([res[2] for res in results])
    sl = torch.cat([res[4] for res in results])
    su = torch.cat([res[5] for res in results])
    return _result(p.n, out, tr, x, theta, sl, su, None, False)


class ShardComm:
    """The NCCL communicator and the fused exchange's IPC-mapped receive
    buffers of one process group, set up once (collectively) and borrowed by
    every sharded solve on it (bx_comm_create / bx_ctx_use_comm): a fresh
    ncclCommInitRank + IPC mapping per solve would cost more than a solve
    step at config 4."""

    def __init__(self, pg, m, exchange):
        import torch.distributed as dist
        L = nat.lib()
        self.m = m
        self.exchange = exchange
        rank, world = dist.get_rank(pg), dist.get_world_size(pg)
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            nat.check(L.bx_nccl_unique_id(uid), None, "bx_nccl_unique_id")
        box = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=pg)
        h = ctypes.c_void_p()
        st = L.bx_comm_create(ctypes.byref(h), box[0], rank, world)
        if st != 0:
            nat.check(st, None, "bx_comm_create")
        self.handle = h
        self.fused = False
        if exchange == "fused":
            # every rank takes part in the gather and the agreement even when
            # its own step failed; any failure puts all ranks on NCCL
            hb = ctypes.create_string_buffer(64)
            ok = L.bx_comm_peer_alloc(h, m, hb) == 0
            hs = [None] * world
            dist.all_gather_object(hs, hb.raw, group=pg)
            ok = ok and L.bx_comm_peer_open(h, b"".join(hs)) == 0
            if agree_all(ok, pg):
                self.fused = True
            else:
                L.bx_comm_peer_disable(h)
                import warnings
                warnings.warn("fused peer exchange unavailable on some rank; using the NCCL schedule")

    def close(self):
        if self.handle:
            nat.lib().bx_comm_destroy(self.handle)
            self.handle = None


_COMMS = {}


def shard_comm(pg, m, exchange):
    """The cached ShardComm of ``pg`` (created on first use, collectively)."""
    import torch.distributed as dist
    key = (id(pg), dist.get_rank(pg), dist.get_world_size(pg), exchange)
    cm = _COMMS.get(key)
    if cm is None or cm.m < m:
        if cm is not None:
            cm.close()
        cm = _COMMS[key] = ShardComm(pg, m, exchange)
    return cm


def release_comms():
    """Destroy the cached communicators (call before destroy_process_group)."""
    for cm in _COMMS.values():
        cm.close()
    _COMMS.clear()


def solve_distributed(p_shard, col_offset, n_global, cfg=None, screening=True, tv=None, loss=QuadraticLoss,
                      slack_scale=None, return_device=True, pg=None, profile=False, exchange=None):
    """This rank's part of an NCCL column-sharded solve (call on every rank of
    the torch.distributed group ``pg``).  Returns the rank-local result: x is
    the shard's block, trace / gap / theta are global.  The communicator is
    created on the first call for ``pg`` and reused (shard_comm)."""
    cfg = cfg or SolverConfig()
    slack_scale = _default_slack(p_shard) if slack_scale is None else slack_scale
    cm = shard_comm(pg, p_shard.m, _exchange(exchange))
    with _Session(p_shard, tv=tv) as s:
        s.use_comm(cm, col_offset, n_global)
        out, tr, x, theta, sl, su = s.run(cfg, screening, loss.alpha, slack_scale, profile=profile)
        prof = s.profile
    return _result(n_global, out, tr, x, theta, sl, su, prof, return_device, n_total=n_global)

"""World-size-2 gloo tests of the column-sharded decomposition on CPU.

The native sharded loop needs a GPU (tests/test_gpu_sharded.py runs it on the
box through the in-process rank group); here two gloo ranks run the sharded
restatement (tests/sharded_oracle.py) with real torch.distributed allreduces
and must reproduce the unsharded oracle round by round."""

import os
import socket

import numpy as np
import pytest


# (config recipe, m, n, rounds): sizes where screening fires inside the window
CASES = {"pg": (1, 100, 200, 1400), "apg": (3, 200, 500, 122)}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        from oracle.boxscreen_oracle import safe_step
        from paper_2202_07258_b200.distributed import column_blocks
        from paper_2202_07258_b200.generate import make_config
        from sharded_oracle import sharded_rounds

        cid, m, n, rounds = CASES[kind]
        inst = make_config(cid, m=m, n=n)

        def allreduce(arr, op):
            t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)
            return t.numpy()

        eta = safe_step(inst.a)
        c0, c1 = column_blocks(inst.a.shape[1], world)[rank]
        tr, x = sharded_rounds(inst.a[:, c0:c1], inst.y, inst.lower[c0:c1], inst.upper[c0:c1], c0,
                               inst.a.shape[1], kind, eta, rounds=rounds, passes=10, allreduce=allreduce)
        xs = [None] * world
        dist.all_gather_object(xs, x)
        if rank == 0:
            q.put((tr, np.concatenate(xs), eta))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["pg", "apg"])
def test_two_rank_gloo_matches_unsharded_oracle(kind):
    import torch.multiprocessing as mp
    from oracle.boxscreen_oracle import oracle_solve
    from paper_2202_07258_b200.generate import make_config
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    tr, x, eta = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cid, m, n, rounds = CASES[kind]
    inst = make_config(cid, m=m, n=n)
    o = oracle_solve(inst.a, inst.y, inst.lower, inst.upper, kind=kind, inner_passes=10, gap_tol=1e-300,
                     max_rounds=rounds, step_size=eta)
    assert len(tr) == len(o["trace"]) == rounds
    assert o["trace"][-1]["preserved"] < n  # screening happened inside the window
    for i, (a, b) in enumerate(zip(tr, o["trace"])):
        scale = max(abs(b["primal"]), abs(b["dual"]), 1e-3)
        for f in ("primal", "dual", "gap"):
            assert abs(a[f] - b[f]) <= 1e-10 * scale, (i, f, a[f], b[f])
        assert a["preserved"] == b["preserved"], (i, a["preserved"], b["preserved"])
    assert np.max(np.abs(x - o["x"])) <= 1e-8 * max(1.0, np.max(np.abs(o["x"])))


def test_column_blocks():
    from paper_2202_07258_b200.distributed import column_blocks
    with pytest.raises(ValueError):
        column_blocks(3, 4)  # every rank needs a column
    for n in (1, 7, 50000):
        for w in (1, 2, 3, 8):
            if n < w:
                continue
            b = column_blocks(n, w)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(c1 - c0 for c0, c1 in b) - min(c1 - c0 for c0, c1 in b) <= 1


def _agree_worker(rank, world, port, oks, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, os.path.dirname(here))
        from paper_2202_07258_b200.distributed import agree_all
        q.put((rank, [agree_all(ok) for ok in oks[rank]]))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_fallback_agreement():
    """The fused peer exchange is used only when every rank mapped its peers
    (distributed.agree_all): one failing rank turns it off on all ranks, so
    every rank runs the same per-step schedule."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    oks = [[True, True, False], [True, False, True]]
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, oks, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] == [True, False, False]

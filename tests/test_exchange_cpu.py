"""The fused reduce + peer-exchange protocol (csrc/bx_exchange.cuh) modelled
on CPU with gloo ranks (world 2 and 3).

Each process stands in for one GPU: its receive buffer and flags live in a
POSIX shared-memory segment (the stand-in for a CUDA IPC allocation), the
segment names travel over torch.distributed (all_gather_object, like the IPC
handles in distributed.solve_distributed), and every rank stores its row
blocks straight into the peers' segments, publishes per-(rank, block) epoch
flags and spins on its own flags -- the kernel's steps 1-5 with the same
buffer layout (2 parities x ranks x payload), the same epoch rule (reached =
v - epoch >= 0 mod 2^32) and rank-order summation.  Random delays between
calls make ranks run ahead of each other.  Checked: no deadlock, every call's
sum is exact and bit-identical on every rank, and a single-buffered variant
(negative control) is caught corrupting data.
"""

import os
import socket
import time

import numpy as np
import pytest

M, NB, EXTRA, CALLS = 96, 3, 8, 60


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _per_cta(m, nb):
    per = (m + nb - 1) // nb
    return (per + 31) // 32 * 32


def _worker(rank, world, port, double_buffer, q):
    import torch.distributed as dist
    from multiprocessing import shared_memory
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pay = M + EXTRA
    nbuf = 2 if double_buffer else 1
    nbytes = nbuf * world * pay * 8 + world * NB * 4
    shm = shared_memory.SharedMemory(create=True, size=nbytes)
    peers = []
    recv = flag = mine_r = mine_f = None
    try:
        shm.buf[:nbytes] = bytes(nbytes)
        names = [None] * world
        dist.all_gather_object(names, shm.name)          # the IPC handle exchange
        for nm in names:
            seg = shm if nm == shm.name else shared_memory.SharedMemory(name=nm)
            peers.append(seg)
        recv = [np.frombuffer(p.buf, dtype=np.float64, count=nbuf * world * pay).reshape(nbuf, world, pay)
                for p in peers]
        flag = [np.frombuffer(p.buf, dtype=np.uint32, count=world * NB, offset=nbuf * world * pay * 8)
                .reshape(world, NB) for p in peers]
        mine_r, mine_f = recv[rank], flag[rank]
        rng = np.random.default_rng(100 + rank)
        per = _per_cta(M, NB)
        bad = 0
        for call in range(1, CALLS + 1):
            epoch = np.uint32(call)
            par = call % nbuf
            local = np.random.default_rng(1000 * call + rank).standard_normal(M)
            # steps 1-3: store every block into every peer, then publish it
            for cta in range(NB):
                r0, r1 = min(M, cta * per), min(M, (cta + 1) * per)
                for p in range(world):
                    recv[p][par, rank, r0:r1] = local[r0:r1]
                for p in range(world):
                    flag[p][rank, cta] = epoch
            # step 4: wait for every peer's blocks (v - epoch >= 0 mod 2^32)
            for cta in range(NB):
                for p in range(world):
                    t0 = time.time()
                    while np.int32(np.uint32(mine_f[p, cta]) - epoch) < 0:
                        if time.time() - t0 > 20:
                            raise RuntimeError("exchange deadlock")
            # step 5: peers in rank order (straggle first so fast ranks run ahead)
            time.sleep(float(rng.uniform(0, 0.004)))
            got = mine_r[par, 0, :M].copy()
            for p in range(1, world):
                got = got + mine_r[par, p, :M]
            want = np.random.default_rng(1000 * call).standard_normal(M)
            for p in range(1, world):
                want = want + np.random.default_rng(1000 * call + p).standard_normal(M)
            bad += int(not np.array_equal(got, want))
        results = [None] * world
        dist.all_gather_object(results, bad)
        dist.barrier()
        if rank == 0:
            q.put(results)
    finally:
        del recv, flag, mine_r, mine_f  # numpy views pin the segments
        for p in peers:
            if p is not shm:
                p.close()
        dist.barrier()
        shm.close()
        shm.unlink()
        dist.destroy_process_group()


def _run(world, double_buffer):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, double_buffer, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_protocol_exact_and_deadlock_free(world):
    assert _run(world, double_buffer=True) == [0] * world


def test_single_buffer_race_is_detected():
    """Negative control: without the parity double buffer a rank that runs
    ahead overwrites the block a slower peer is still summing."""
    res = _run(2, double_buffer=False)
    assert sum(res) > 0

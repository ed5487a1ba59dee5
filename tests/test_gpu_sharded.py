"""Column-sharded solves on one GPU through the in-process rank
group: the exact native code path of the NCCL build (phase-A partial rows ->
allreduce -> phase-B objective, epsilon MAX, bound-term SUM, global counts,
global power iteration), compared with the single-context solve."""

import numpy as np
import pytest

from conftest import small_instance
from parity import compare_final, compare_traces

pytestmark = pytest.mark.gpu


def _oracle_like(res):
    """Adapt a GPU SolveResult to the oracle-dict shape parity.py compares."""
    return dict(trace=[dict(primal=t.primal, dual=t.dual, gap=t.gap, preserved=t.preserved_count)
                       for t in res.trace],
                x=np.asarray(res.x), sat_lower=np.asarray(res.sat_lower), sat_upper=np.asarray(res.sat_upper),
                converged=res.converged)


@pytest.mark.parametrize("exchange", ["fused", "nccl"])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("cfg_id,kind,m,n", [(3, "apg", 1000, 5000), (1, "pg", 600, 1500)])
def test_sharded_matches_single(nranks, cfg_id, kind, m, n, exchange):
    """exchange="fused": the per-step reduction as the fused reduce + peer
    exchange kernel (all ranks in one cooperative launch on this GPU);
    "nccl": the collective schedule through the group's allreduce."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.distributed import solve_group
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(cfg_id, m=m, n=n)
    p = Problem(inst.a, inst.y, inst.lower, inst.upper)
    cfg = SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-6, max_rounds=400)
    single = solve(p, cfg)
    sh = solve_group(p, cfg, nranks=nranks, exchange=exchange)
    probs = compare_traces(sh, _oracle_like(single)) + compare_final(sh, _oracle_like(single))
    assert not probs, probs[:3]


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_production_exchange_kernel_per_rank(nranks, dtype, monkeypatch):
    """The production ``k_xreduce`` -- one launch per rank on the rank's own
    stream, 2 and 4 co-resident grids exchanging through the peer buffers and
    epoch flags (bounded waits: a protocol error would surface as PeerTimeout,
    not a hang) -- against the one-launch group kernel: every rank's trace
    bit-identical, run after run, and equal to the single-context trajectory."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.distributed import solve_group
    from paper_2202_07258_b200.generate import make_config
    monkeypatch.setenv("BX_PEER_TIMEOUT_S", "10")
    inst = make_config(3, m=1000, n=5000)
    p = Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=dtype)
    cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=120)
    peer = solve_group(p, cfg, nranks=nranks, exchange="peer", return_shards=True)
    fused = solve_group(p, cfg, nranks=nranks, exchange="fused", return_shards=True)
    for r in range(nranks):
        for f in ("primal", "dual", "gap", "preserved_count"):
            np.testing.assert_array_equal(peer[r][1][f], peer[0][1][f])
            np.testing.assert_array_equal(peer[r][1][f], fused[r][1][f])
    if dtype is np.float64:
        single = solve(p, cfg)
        sh = solve_group(p, cfg, nranks=nranks, exchange="peer")
        probs = compare_traces(sh, _oracle_like(single)) + compare_final(sh, _oracle_like(single))
        assert not probs, probs[:3]


def test_fused_exchange_is_deterministic_and_rank_consistent():
    """Every rank sums the peers' blocks in rank order: identical residual
    bits on every rank (same trace from every shard) and run to run; the
    fp32-storage pass goes through the same kernel."""
    from paper_2202_07258_b200 import Problem, SolverConfig
    from paper_2202_07258_b200.distributed import solve_group
    from paper_2202_07258_b200.generate import make_config
    inst = make_config(3, m=800, n=4000)
    for dt in (np.float64, np.float32):
        p = Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=dt)
        cfg = SolverConfig(kind="apg", inner_passes=10, gap_tol=1e-6, max_rounds=60)
        runs = [solve_group(p, cfg, nranks=4, return_shards=True) for _ in range(2)]
        for shards in runs:
            ref = shards[0][1]
            for other in shards[1:]:
                for f in ("primal", "dual", "gap", "preserved_count"):
                    np.testing.assert_array_equal(other[1][f], ref[f])
        for f in ("primal", "gap"):
            np.testing.assert_array_equal(runs[0][0][1][f], runs[1][0][1][f])


@pytest.mark.parametrize("family", ["bvls", "mixed"])
def test_sharded_bound_families(family):
    """Nonzero bounds exercise the replicated z update; mixed bounds with
    contiguous blocks leave some ranks without infinite uppers (global eps)."""
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    from paper_2202_07258_b200.distributed import solve_group
    rng = np.random.default_rng(77)
    for _ in range(3):
        n = int(rng.integers(12, 40))
        m = int(rng.integers(n, 80))
        a, y, lo, hi = small_instance(rng, m, n, family)
        if family == "mixed":
            hi[: n // 2] = rng.uniform(0.2, 2.0, n // 2)   # first block all finite
            hi[n // 2:] = np.inf
        p = Problem(a, y, lo, hi)
        for kind in ("pg", "apg"):
            cfg = SolverConfig(kind=kind, inner_passes=10, gap_tol=1e-8)
            single = solve(p, cfg)
            sh = solve_group(p, cfg, nranks=2)
            probs = compare_traces(sh, _oracle_like(single)) + compare_final(sh, _oracle_like(single))
            assert not probs, (family, kind, probs[:3])


def test_sharded_cd_is_rejected():
    from paper_2202_07258_b200 import Problem, SolverConfig
    from paper_2202_07258_b200.distributed import solve_group
    from paper_2202_07258_b200.errors import NativeError
    rng = np.random.default_rng(1)
    a, y, lo, hi = small_instance(rng, 20, 10, "bvls")
    with pytest.raises(NativeError):
        solve_group(Problem(a, y, lo, hi), SolverConfig(kind="cd"), nranks=2)


def test_nccl_plumbing_under_torchrun():
    """NCCL transport (dlopen'd libnccl, unique-id broadcast, in-place
    allreduce on the context stream) through torchrun with one GPU: the
    collective code path runs with one rank and must reproduce solve()."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "scripts", "nccl_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "OK" in out.stdout

"""Batched many-RHS FISTA on fp64 tensor cores (config 5) vs the batched
oracle (oracle/batched_oracle.py), per problem and per round."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _instance(m, n, K, seed=3):
    rng = np.random.default_rng(seed)
    a = np.abs(rng.standard_normal((m, n))) + 0.05
    X0 = np.zeros((n, K))
    for k in range(K):
        sup = rng.choice(n, size=4, replace=False)
        X0[sup, k] = rng.random(4)
    Y = a @ X0 + 0.05 * rng.standard_normal((m, K))
    return a, Y


@pytest.mark.parametrize("m,n,K,rounds", [(40, 120, 128, 6), (40, 120, 128, 25), (37, 250, 70, 12)])
def test_batched_matches_oracle(m, n, K, rounds):
    from oracle.batched_oracle import batched_apg
    from paper_2202_07258_b200.batched import solve_batched
    a, Y = _instance(m, n, K)
    g = solve_batched(a, Y, passes=10, rounds=rounds, gap_tol=1e-300)
    o = batched_apg(a, Y, eta=g.eta, inner_passes=10, rounds=rounds, gap_tol=1e-300)
    assert g.rounds == rounds
    scale = np.maximum(np.maximum(np.abs(o["primal"][-1]), np.abs(o["dual"][-1])), 1e-3)
    for name, gv in (("primal", g.primal), ("dual", g.dual), ("gap", g.gap)):
        d = np.abs(gv - o[name][-1])
        assert np.all(d <= 1e-10 * scale), (name, d.max(), np.argmax(d / scale))
    np.testing.assert_array_equal(g.preserved, o["preserved"][-1])
    assert np.max(np.abs(g.x - o["X"])) <= 1e-8 * max(1.0, np.abs(o["X"]).max())


def test_batched_screening_on_off_same_optimum():
    """Screening is safe: with and without it every problem reaches the same
    objective (acceptance criterion 2 of the reference, test_acceptance.py:91-100)."""
    from paper_2202_07258_b200.batched import solve_batched
    a, Y = _instance(60, 40, 64, seed=5)          # m > n: strongly convex problems
    on = solve_batched(a, Y, passes=10, rounds=400, gap_tol=1e-10)
    off = solve_batched(a, Y, passes=10, rounds=400, gap_tol=1e-10, screening=False)
    assert on.converged == 64 and off.converged == 64
    assert on.preserved.mean() < 40                 # screening fired
    np.testing.assert_allclose(on.primal, off.primal, rtol=1e-8, atol=1e-12)
    # screened coordinates sit at the bound in the unscreened solution
    assert np.all(np.abs(off.x[on.x == 0.0]) < 1e-6)


def test_bump_dictionary_config5_shape():
    """Config 5 recipe at reduced K: runs, DMMA path, gaps decrease."""
    from paper_2202_07258_b200.batched import solve_batched
    from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
    a = bump_dictionary(200, 5000)
    Y, _ = batched_rhs(a, 256)
    g = solve_batched(a, Y, passes=10, rounds=4, gap_tol=1e-6)
    assert g.rounds == 4
    assert g.trace[-1, 2] < g.trace[0, 2]   # mean gap decreased


def test_sphere_sweep_bound_is_exact(monkeypatch):
    """The per-problem bound of the dual sweep (min_j v_j - eps max|a_j't| +
    thr min||a_j|| > 0: nothing can be screened) only skips sweeps that screen
    nothing: with the bound switched off (BX_BT_NOSKIP=1, every tile runs the
    per-coordinate test) every trace value, mask count and x is bit-identical
    -- on an instance that screens (the sweep must run) and on the config-5
    dictionary (the bound clears every tile)."""
    from paper_2202_07258_b200.batched import solve_batched
    from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
    a, Y = _instance(60, 40, 128, seed=5)
    on = solve_batched(a, Y, passes=10, rounds=60, gap_tol=1e-300)
    assert on.preserved.mean() < 40 and on.sphere_sweeps > 0          # screening fired through the sweep
    ab = bump_dictionary(200, 5000)
    Yb, _ = batched_rhs(ab, 128)
    onb = solve_batched(ab, Yb, passes=10, rounds=3, gap_tol=1e-6)
    assert onb.sphere_sweeps == 0 and onb.tiles == 2                   # cleared by the bound
    monkeypatch.setenv("BX_BT_NOSKIP", "1")
    off = solve_batched(a, Y, passes=10, rounds=60, gap_tol=1e-300)
    offb = solve_batched(ab, Yb, passes=10, rounds=3, gap_tol=1e-6)
    assert off.sphere_sweeps == 60 * off.tiles and offb.sphere_sweeps == 3 * offb.tiles
    for u, v in ((on, off), (onb, offb)):
        for f in ("primal", "dual", "gap", "preserved"):
            np.testing.assert_array_equal(getattr(u, f), getattr(v, f))
        np.testing.assert_array_equal(u.x, v.x)


def test_result_streamed_to_host_during_last_round():
    """More tiles than SMs: the last round of the budget runs wave by wave and
    each wave's columns of X are copied to the (pinned) host buffer while the
    next waves compute (bx_batched_run_to_host); same bits as the device
    result, also when the solve stops before the budget (copy after the last
    round) and into a caller-supplied buffer."""
    import torch
    from paper_2202_07258_b200.batched import solve_batched
    K = 149 * 64 + 7
    a, Y = _instance(16, 40, K, seed=11)
    dev = solve_batched(a, Y, passes=10, rounds=3, gap_tol=1e-300, return_device=True)
    host = solve_batched(a, Y, passes=10, rounds=3, gap_tol=1e-300)
    np.testing.assert_array_equal(host.x, dev.x.cpu().numpy())
    np.testing.assert_array_equal(host.gap, dev.gap)
    buf = torch.empty((K, 40), dtype=torch.float64, pin_memory=True)
    early = solve_batched(a, Y, passes=10, rounds=50, gap_tol=1e30, x_out=buf)      # converged after round 1
    assert early.rounds == 1
    one = solve_batched(a, Y, passes=10, rounds=1, gap_tol=1e-300, return_device=True)
    np.testing.assert_array_equal(early.x, one.x.cpu().numpy())
    with pytest.raises(ValueError):
        solve_batched(a, Y, passes=10, rounds=1, x_out=torch.empty((K, 40), dtype=torch.float64))


@pytest.mark.parametrize("m,n,K,check_every", [(40, 120, 192, 4), (37, 250, 70, 16), (16, 40, 149 * 64 + 7, 3)])
def test_rounds_overlapping_across_a_launch(m, n, K, check_every):
    """check_every > 1: one launch runs several rounds and a tile's next round
    starts as soon as its own previous round is done (per-octet flags), on
    whichever SM is free.  Same arithmetic per problem, so every trace row,
    every per-problem value and x are bit-identical to one launch per round --
    with fewer tiles than SMs, with more (units wrap around the grid), and
    with the result streamed to the host."""
    from paper_2202_07258_b200.batched import solve_batched
    a, Y = _instance(m, n, K, seed=21)
    rounds = 11
    one = solve_batched(a, Y, passes=10, rounds=rounds, gap_tol=1e-300)
    many = solve_batched(a, Y, passes=10, rounds=rounds, gap_tol=1e-300, check_every=check_every)
    assert many.rounds == one.rounds == rounds
    np.testing.assert_array_equal(many.trace, one.trace)
    for f in ("primal", "dual", "gap", "eps", "preserved"):
        np.testing.assert_array_equal(getattr(many, f), getattr(one, f))
    np.testing.assert_array_equal(many.x, one.x)
    odd = solve_batched(a, Y, passes=3, rounds=5, gap_tol=1e-300, check_every=2, return_device=True)   # odd passes: buffer parity per round
    ref = solve_batched(a, Y, passes=3, rounds=5, gap_tol=1e-300, return_device=True)
    np.testing.assert_array_equal(odd.x.cpu().numpy(), ref.x.cpu().numpy())

"""The batched oracle (oracle/batched_oracle.py, which DEFINES config 5's
semantics: the reference has no many-right-hand-side solver) against the
single-problem oracle that is pinned bit for bit to the reference
(oracle/boxscreen_oracle.py, tests/test_oracle.py): run problem by problem
with the same fixed step, the single-problem FISTA -- compaction, reduced dual
point -- must take the same screening decisions and reach the same objectives
as the batched formulation -- masks, full-problem dual point.  CPU only."""

import numpy as np
import pytest

from oracle.batched_oracle import batched_apg, power_step
from oracle.boxscreen_oracle import oracle_solve


def _instance(m, n, K, seed):
    rng = np.random.default_rng(seed)
    a = np.abs(rng.standard_normal((m, n))) + 0.05
    X0 = np.zeros((n, K))
    for k in range(K):
        sup = rng.choice(n, size=4, replace=False)
        X0[sup, k] = rng.random(4)
    return a, a @ X0 + 0.05 * rng.standard_normal((m, K))


@pytest.mark.parametrize("m,n,K,rounds,screening", [(40, 30, 6, 12, False), (60, 40, 6, 60, True),
                                                    (25, 50, 4, 40, True)])
def test_batched_oracle_equals_single_problem_oracle(m, n, K, rounds, screening):
    a, Y = _instance(m, n, K, seed=5)
    eta = power_step(a)
    b = batched_apg(a, Y, eta=eta, inner_passes=10, rounds=rounds, gap_tol=1e-300, screening=screening)
    screened_something = False
    for k in range(K):
        o = oracle_solve(np.asfortranarray(a), Y[:, k], np.zeros(n), np.full(n, np.inf), kind="apg",
                         inner_passes=10, gap_tol=1e-300, max_rounds=rounds, screening=screening, step_size=eta)
        tr = o["trace"]
        assert len(tr) == rounds and all(t["step"] == eta for t in tr)      # the step is never re-estimated
        P = np.array([t["primal"] for t in tr])
        pres = np.array([t["preserved"] for t in tr])
        np.testing.assert_array_equal(pres, b["preserved"][:, k])           # identical screening decisions
        assert np.max(np.abs(P - b["primal"][:, k]) / np.maximum(1e-3, np.abs(P))) <= 1e-12
        assert np.max(np.abs(o["x"] - b["X"][:, k])) <= 1e-10 * max(1.0, np.abs(o["x"]).max())
        screened_something |= pres[-1] < n
    assert screened_something == screening or not screening

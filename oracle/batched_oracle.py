"""CPU oracle for the batched many-right-hand-side FISTA (BASELINE config 5).

TEST INFRASTRUCTURE ONLY (same rules as oracle/boxscreen_oracle.py: used by
tests/, smoke() and bench.py's CPU legs, never by the product package).

The reference has no batched solver; this file DEFINES the semantics the GPU
path implements ("Batched FISTA"): K independent NNLS problems
min_x 0.5||y_k - A x||^2, x >= 0 sharing one dictionary A, each run with the
``apg`` iteration of oracle/boxscreen_oracle.py (same momentum, same
function + gradient restart tests with round-off-sized slacks) and its own
Gap-safe screening, with two batched simplifications:

* one step size for all problems, eta = 0.99 / (sigma/0.999)^2 from the power
  iteration on the full A (solvers.py:89-98); it is never re-estimated
  (a smaller preserved set only makes it more conservative);
* screening masks instead of compaction: a screened coordinate of problem k
  is fixed at its bound (0) and frozen; the dual point and the gap are those
  of the FULL problem (epsilon over all columns, duality.py:187-209), so each
  round's gap is already the certified one.

Per round (inner_passes FISTA steps, then the dual point at x):
    v_k = A'theta0_k with theta0_k = y_k - A x_k ; eps_k = max_j (v_jk)+ / |a_j't|
    theta_k = theta0_k + eps_k t ; D_k = theta_k . y_k - 0.5 ||theta_k||^2
    gap_k = max(P_k - D_k, 0) ; r_k = sqrt(2 gap_k) ; slack_k = 1e-12 max(1, ||theta_k||)
    screen j for problem k when v_jk + eps_k a_j't < -(r_k + slack_k) ||a_j||
Problems whose gap is below gap_tol are converged; the batch stops when all are.
"""


import numpy as np

RESTART_SLACK = 1e-12
SLACK_SCALE = 1e-12


def power_step(a, iters=50, seed=0):
    v = np.random.default_rng(seed).standard_normal(a.shape[1])
    v /= np.linalg.norm(v)
    s = 0.0
    for _ in range(iters):
        w = a.T @ (a @ v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 1.0
        v = w / nw
        s = np.sqrt(nw)
    s = s / 0.999
    return 0.99 / s ** 2


def batched_apg(a, Y, eta=None, inner_passes=10, rounds=10, gap_tol=1e-6, screening=True, record=True):
    """Run ``rounds`` rounds on all K = Y.shape[1] problems.  Returns a dict with
    X (n, K), per-round arrays primal/dual/gap (rounds, K), preserved counts
    (rounds, K), converged flags, the final momentum and mask."""
    a = np.asarray(a, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    m, n = a.shape
    K = Y.shape[1]
    eta = power_step(a) if eta is None else eta
    t = -np.ones(m)
    att = a.T @ t
    nrm = np.linalg.norm(a, axis=0)
    X = np.zeros((n, K))
    Xp = np.zeros((n, K))
    R = a @ X - Y
    Rp = R.copy()
    mom = np.ones(K)
    P = 0.5 * np.sum(R * R, axis=0)
    active = np.ones((n, K), dtype=bool)
    conv = np.zeros(K, dtype=bool)
    hist = dict(primal=[], dual=[], gap=[], preserved=[])
    for _ in range(rounds):
        for _ in range(inner_passes):
            tn = (1.0 + np.sqrt(1.0 + 4.0 * mom * mom)) / 2.0
            beta = (mom - 1.0) / tn
            Yv = X + beta * (X - Xp)
            Ry = R + beta * (R - Rp)
            G = a.T @ Ry
            Xn = np.where(active, np.maximum(Yv - eta * G, 0.0), 0.0)
            Rn = a @ Xn - Y
            Pn = 0.5 * np.sum(Rn * Rn, axis=0)
            dX = Xn - X
            gdot = np.sum(G * dX, axis=0)
            s_f = RESTART_SLACK * np.maximum(1.0, np.abs(P))
            s_g = RESTART_SLACK * np.sqrt(2.0 * P) * (nrm @ np.abs(dX))
            restart = (Pn > P + s_f) | (gdot > s_g)
            Xp, Rp = X, R
            X, R = Xn, Rn
            mom = np.where(restart, 1.0, tn)
            P = Pn
        # dual point of the full problem at x (NNLS, t = -1)
        V = -(a.T @ R)
        eps = np.max(np.maximum(V, 0.0) / np.abs(att)[:, None], axis=0)
        theta = -R + eps[None, :] * t[:, None]
        V = V + eps[None, :] * att[:, None]
        D = np.sum(theta * Y, axis=0) - 0.5 * np.sum(theta * theta, axis=0)
        gap = np.maximum(P - D, 0.0)
        P_gap = P.copy()
        conv = gap < gap_tol
        if screening:
            radius = np.sqrt(2.0 * gap)
            slack = SLACK_SCALE * np.maximum(1.0, np.sqrt(np.sum(theta * theta, axis=0)))
            new = active & (V < -(radius + slack)[None, :] * nrm[:, None])
            if new.any():
                active &= ~new
                X = np.where(active, X, 0.0)
                Xp = np.where(active, Xp, 0.0)
                R = a @ X - Y
                Rp = a @ Xp - Y
                P = 0.5 * np.sum(R * R, axis=0)
        if record:
            hist["primal"].append(P_gap)
            hist["dual"].append(D.copy())
            hist["gap"].append(gap.copy())
            hist["preserved"].append(active.sum(axis=0))
        if conv.all():
            break
    return dict(X=X, converged=conv, mom=mom, active=active, eta=eta,
                **{k: np.array(v) for k, v in hist.items()})

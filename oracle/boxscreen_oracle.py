"""CPU oracle for the screened box-constrained least-squares iteration.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(``paper_2202_07258_b200``) imports, calls or links this module.  It may be
used by ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` -- always as the checker or as the
timed CPU baseline, never as the measured or shipped path.

What it is: a numpy restatement of the reference ``boxscreen`` package's
Algorithm-1 loop (Dantas, Soubies, Fevotte, arXiv 2202.07258), restricted to
the hot path named by ``BASELINE.json:north_star``:

* projected gradient ``pg``      -- /root/reference/pkg/src/boxscreen/solvers.py:101-116
* cyclic coordinate descent ``cd`` -- solvers.py:119-137
* the preserved-column workspace -- solvers.py:48-69
* power-iteration step rule      -- solvers.py:72-98
* dual translation / scaling, reduced dual, gap clamp, certified gap
                                 -- driver.py:183-209, 112-128; duality.py:103-209
* bounded-variable active set (Lawson-Hanson) ``active-set``
                                 -- solvers.py:140-204 (+ ActiveSetState, :38-45;
                                    x0 = l and 10 n rounds, driver.py:144-147;
                                    KKT-optimal exit, driver.py:246-252)
* gap-safe sphere test + slack   -- screening.py:11-15, 46-69; driver.py:214-221
* screening application / compaction / step re-estimate
                                 -- screening.py:72-94; driver.py:222-235

Extensions the reference does not contain (BASELINE.json configs 3 and 5),
defined here in the same workspace/round conventions and documented in
DESIGN.md ("FISTA definition"):

* ``apg`` -- FISTA momentum with restart on an objective increase (plus, by
  default, the O'Donoghue-Candes gradient test), the extrapolated gradient
  carried by linearity (g(y) = g + beta (g - g_prev)), momentum kept across
  screening events with g_prev recomputed on the compacted set.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(imported from /root/reference in the build container) on seeded instances
and stores its per-round traces and final states; ``tests/test_oracle.py``
checks this restatement reproduces them bit for bit (pg, cd).  The ``apg``
extension is pinned only at solution level (objective equal to the
reference's high-accuracy optimum within the cross-solver tolerance
test_solvers.py:205, screened coordinates saturated in that optimum).
"""

import math

import numpy as np
import scipy.linalg as sla

GAP_ROUNDOFF = 1e-9          # duality.py:24 (weak-duality round-off slack)
SLACK_SCALE = 1e-12          # driver.py:219
INTERIOR_TOL = 1e-10         # duality.py:48 (strict_tol)
RESTART_SLACK = 1e-12        # FISTA restart threshold (extension)


class OracleError(Exception):
    """Raised with ``kind`` set to the reference exception class name."""

    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# setup-time quantities
# --------------------------------------------------------------------------

def column_norms(a):
    """||a_j||_2 per column (model.py:89-92)."""
    return np.linalg.norm(a, axis=0)


def spectral_sigma(a, iters=50, seed=0):
    """Power iteration on A'A from a seeded Gaussian start (solvers.py:72-86)."""
    start = np.random.default_rng(seed).standard_normal(a.shape[1])
    v = start / np.linalg.norm(start)
    s = 0.0
    for _ in range(iters):
        w = a.T @ (a @ v)
        nrm = np.linalg.norm(w)
        if nrm == 0.0:
            return 0.0
        v = w / nrm
        s = np.sqrt(nrm)
    return float(s)


def safe_step(a, alpha=1.0, iters=50):
    """eta = 0.99 alpha / (sigma/0.999)^2, or 1 for a zero matrix (solvers.py:89-98)."""
    s = spectral_sigma(a, iters) / 0.999
    if s == 0.0:
        return 1.0
    return 0.99 * alpha / s ** 2


def translation_att(a, t, norms):
    """A't with the strict-interiority check (duality.py:48-59)."""
    att = a.T @ t
    if np.any(att >= -INTERIOR_TOL * norms):
        raise OracleError("NoInteriorPoint", f"max a_j't = {att.max():.3e}")
    return att


def clamp(gap):
    """duality.py:152-156."""
    if gap < -GAP_ROUNDOFF:
        raise OracleError("InternalConsistency", f"duality gap {gap:.3e}")
    return max(gap, 0.0)


# --------------------------------------------------------------------------
# the full-problem certificate (driver.py:112-117 -> duality.py:159-209)
# --------------------------------------------------------------------------

def certified_gap(a, y, lo, hi, inf_mask, x, t=None, att=None):
    ax = a @ x
    zg = -(ax - y)
    atz = a.T @ zg
    if inf_mask.any():
        eps = float(np.max(np.maximum(atz[inf_mask], 0.0) / np.abs(att[inf_mask])))
        theta = zg + eps * t
        atth = atz + eps * att
    else:
        theta = zg
        atth = atz
    # dual objective (duality.py:103-124) with the quadratic conjugate
    u = -theta
    d = -float(np.sum(u * y + 0.5 * u * u))
    d -= float(lo @ np.minimum(atth, 0.0))
    fin = ~inf_mask
    if fin.any():
        d -= float(hi[fin] @ np.maximum(atth[fin], 0.0))
    res = ax - y
    primal = 0.5 * float(res @ res)
    return clamp(primal - d), theta, primal, d


# --------------------------------------------------------------------------
# the preserved-column view (solvers.py:48-69)
# --------------------------------------------------------------------------

class ActiveView:
    def __init__(self, a, y, lo, hi, norms, z, x_full, keep):
        self.idx = keep
        self.mat = np.asfortranarray(a[:, keep])
        self.lo = lo[keep]
        self.hi = hi[keep]
        self.sq = norms[keep] ** 2
        self.nrm = norms[keep]
        self.x = x_full[keep].copy()
        self.off = z - y            # A x + off  = residual
        self.tgt = y - z            # reduced-problem target
        self.r = self.mat @ self.x + self.off
        self.g = self.mat.T @ self.r
        # apg state (not part of the reference workspace): previous iterate
        # and the gradient there
        self.x_prev = None
        self.g_prev = None

    def write_back(self, x_full):
        x_full[self.idx] = self.x


# --------------------------------------------------------------------------
# primal updates
# --------------------------------------------------------------------------

def pg_passes(w, eta, passes):
    """solvers.py:101-116."""
    obj = 0.5 * float(w.r @ w.r)
    for _ in range(passes):
        w.x = np.clip(w.x - eta * w.g, w.lo, w.hi)
        w.r = w.mat @ w.x + w.off
        nobj = 0.5 * float(w.r @ w.r)
        if nobj > obj + 1e-9:
            raise OracleError("StepSizeTooLarge", f"objective rose {obj:.6e} -> {nobj:.6e}")
        obj = nobj
        w.g = w.mat.T @ w.r


def cd_passes(w, passes):
    """solvers.py:119-137 (exact per-coordinate minimisation, original order)."""
    x, r, mat, lo, hi, sq = w.x, w.r, w.mat, w.lo, w.hi, w.sq
    for _ in range(passes):
        for k in range(x.size):
            col = mat[:, k]
            s = float(col @ r) / sq[k]
            nv = min(max(x[k] - s, lo[k]), hi[k])
            d = nv - x[k]
            if d != 0.0:
                r += d * col
                x[k] = nv
    w.g = mat.T @ r


def apg_passes(w, eta, passes, mom, restart="adaptive"):
    """FISTA extension (not in the reference; see module docstring).

    ``mom`` is a one-element list holding the momentum scalar t_k (t=1 means
    no extrapolation on the next step).  ``w.g`` is the gradient A'r at the
    current x (the Workspace invariant, solvers.py:65-69) and ``w.g_prev``
    the gradient at the previous iterate.  Per step:
        t' = (1 + sqrt(1 + 4 t^2)) / 2 ;  beta = (t - 1) / t'
        y  = x + beta (x - x_prev) ;  g_y = g + beta (g - g_prev)
                                      (= A'r(y): the gradient is affine in x)
        x+ = clip(y - eta g_y, lo, hi) ;  r+ = A x+ + off ;  g+ = A'r+
        restart (t <- 1) when  P(x+) > P(x) + s_f      (objective increase,
                                                       the BASELINE config-3 rule)
                           or  g_y'(x+ - x) > s_g      (gradient test of
                                                       O'Donoghue & Candes 2015;
                                                       restart="adaptive" only)
        otherwise t <- t'.  Slacks sized to each test's own round-off, so
        the CPU oracle and the GPU (different summation orders) agree:
            s_f = 1e-12 max(1, P(x))                        (noise in P ~1e-14 P)
            s_g = 1e-12 ||r|| sum_j ||a_j|| |x+_j - x_j|    (noise in g_j ~ eps ||a_j|| ||r||)
    Each step reads A twice, like pg_step (solvers.py:109-116): A x+ and
    A'r+.  The gradient at the new iterate is the one the next step, and the
    round's dual point (driver.py:183-198), both need -- so the GPU streams A
    once per step and evaluates the round's dual point from the first pass of
    the next round ("speculative round boundary").
    The gradient test keeps restarting deep in the tail, where objective
    changes are far below s_f; without it the momentum grows unbounded and
    FISTA degrades to its O(1/k^2) regime ("FISTA definition").
    """
    obj = 0.5 * float(w.r @ w.r)
    if w.x_prev is None:
        w.x_prev = w.x.copy()
        w.g_prev = w.g.copy()
    for _ in range(passes):
        t = mom[0]
        tn = (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
        beta = (t - 1.0) / tn
        if beta != 0.0:
            yv = w.x + beta * (w.x - w.x_prev)
            gy = w.g + beta * (w.g - w.g_prev)
        else:
            yv = w.x
            gy = w.g
        xn = np.clip(yv - eta * gy, w.lo, w.hi)
        rn = w.mat @ xn + w.off
        nobj = 0.5 * float(rn @ rn)
        dx = xn - w.x
        gdot = float(gy @ dx)
        s_f = RESTART_SLACK * max(1.0, abs(obj))
        s_g = RESTART_SLACK * math.sqrt(2.0 * obj) * float(w.nrm @ np.abs(dx))
        w.x_prev, w.g_prev = w.x, w.g
        w.x, w.r = xn, rn
        w.g = w.mat.T @ w.r
        grad_test = restart == "adaptive" and gdot > s_g
        mom[0] = 1.0 if (nobj > obj + s_f or grad_test) else tn
        obj = nobj


def _passive_lstsq(mat, rhs, cols):
    """Least squares on the passive columns through the Cholesky factor of
    their Gram matrix (solvers.py:140-148; the same LAPACK calls, so the
    restatement reproduces the reference bit for bit)."""
    sub = mat[:, cols]
    try:
        fac = sla.cho_factor(sub.T @ sub)
    except sla.LinAlgError:
        raise OracleError("SingularSubproblem", "passive-column least-squares system is singular")
    return sla.cho_solve(fac, sub.T @ rhs)


def active_set_pass(w, passive):
    """One outer bounded-variable Lawson-Hanson iteration (solvers.py:151-204).

    ``passive`` (bool over the view's columns) is updated in place.  Returns
    True when no bound coordinate violates the optimality conditions.
    """
    x, lo, hi = w.x, w.lo, w.hi
    neg_g = -w.g
    tol = 1e-10 * w.nrm * max(float(np.linalg.norm(w.r)), 1.0)
    bound = ~passive
    pull_up = bound & (x <= lo) & (neg_g > tol)
    pull_dn = bound & ~np.isinf(hi) & (x >= hi) & (neg_g < -tol)
    score = np.maximum(np.where(pull_up, neg_g, 0.0), np.where(pull_dn, -neg_g, 0.0))
    if not score.any():
        return True
    passive[int(np.argmax(score))] = True
    for _ in range(2 * x.size + 2):
        free = np.flatnonzero(passive)
        fixed = ~passive
        rhs = w.tgt - w.mat[:, fixed] @ x[fixed] if fixed.any() else w.tgt
        s = _passive_lstsq(w.mat, rhs, free)
        lo_f, hi_f = lo[free], hi[free]
        low, high = s < lo_f, s > hi_f
        if not (low.any() or high.any()):
            x[free] = s
            break
        cur = x[free]
        with np.errstate(divide="ignore", invalid="ignore"):
            frac = np.where(low, (lo_f - cur) / (s - cur),
                            np.where(high, (hi_f - cur) / (s - cur), np.inf))
        step = min(max(float(np.min(frac)), 0.0), 1.0)
        x[free] = cur + step * (s - cur)
        hit = frac <= step + 1e-12
        x[free[hit & low]] = lo_f[hit & low]
        x[free[hit & high]] = hi_f[hit & high]
        passive[free[hit]] = False
    else:
        raise OracleError("SingularSubproblem", "active-set inner loop failed to make progress")
    w.r = w.mat @ x + w.off
    w.g = w.mat.T @ w.r
    return False


# --------------------------------------------------------------------------
# Algorithm 1 (driver.py:131-256)
# --------------------------------------------------------------------------

def oracle_solve(a, y, lo, hi, kind="pg", inner_passes=1, gap_tol=1e-6,
                 max_rounds=None, screening=True, step_size=None, t=None,
                 power_iters=50, record_sets=False, round_hook=None, restart="adaptive", init=None):
    """Run the screened solver and return a dict with x, theta, gap, rounds,
    converged, trace (list of per-round dicts), sat_lower, sat_upper.

    ``a`` must be an fp64 (m, n) array; Fortran order is used internally.
    Per-round trace entries carry primal, dual, gap, eps, radius, slack,
    preserved count, newly screened counts and (with ``record_sets``) the
    newly screened index arrays; ``step`` is the step in force.

    ``init`` resumes mid-solve from a given state (replaying rounds from a
    device solve's state, tests/test_gpu_headline.py): dict(x, sat_lower,
    sat_upper, eta, basis, round0 [, x_prev, mom for apg]); x holds the
    screened coordinates at their bounds, the preserved set is the
    complement of the saturated sets in original order, z = A_S b_S.
    """
    a = np.asarray(a, dtype=float, order="F")
    y = np.asarray(y, dtype=float).ravel()
    m, n = a.shape
    lo = np.broadcast_to(np.asarray(lo, dtype=float), (n,)).copy()
    hi = np.broadcast_to(np.asarray(hi, dtype=float), (n,)).copy()
    inf_mask = np.isinf(hi)
    norms = column_norms(a)
    att_full = None
    if inf_mask.any():
        # the translation vector is built before the screening state
        # (driver.py:141-152), so NoInteriorPoint precedes ZeroColumn
        t = -np.ones(m) if t is None else np.asarray(t, dtype=float).ravel()
        att_full = translation_att(a, t, norms)
    if np.any(norms == 0.0):
        raise OracleError("ZeroColumn", f"zero column at {int(np.argmin(norms))}")
    if kind not in ("pg", "cd", "apg", "active-set"):
        raise ValueError(kind)
    if kind == "active-set":
        # coordinates start on a bound (driver.py:144-147)
        x_full = lo.copy()
        limit = max_rounds or 10 * n
        passive_full = np.zeros(n, dtype=bool)
    else:
        x_full = np.clip(np.zeros(n), lo, hi)
        limit = max_rounds or 10 ** 6
    keep = np.arange(n)
    sat_lo = np.empty(0, dtype=int)
    sat_up = np.empty(0, dtype=int)
    z = np.zeros(m)
    eta = step_size
    basis = n
    round0 = 0
    mom = [1.0]
    if init is not None:
        x_full = np.asarray(init["x"], dtype=float).copy()
        sat_lo = np.asarray(init["sat_lower"], dtype=int).copy()
        sat_up = np.asarray(init["sat_upper"], dtype=int).copy()
        keep = np.setdiff1d(np.arange(n), np.concatenate([sat_lo, sat_up]))
        if sat_lo.size:
            z = z + a[:, sat_lo] @ lo[sat_lo]
        if sat_up.size:
            z = z + a[:, sat_up] @ hi[sat_up]
        eta = float(init["eta"])
        basis = int(init["basis"])
        round0 = int(init.get("round0", 0))
        mom = [float(init.get("mom", 1.0))]
    if kind in ("pg", "apg") and eta is None:
        eta = safe_step(a, 1.0, power_iters)
    w = ActiveView(a, y, lo, hi, norms, z, x_full, keep)
    if init is not None and kind == "apg" and init.get("x_prev") is not None:
        w.x_prev = np.asarray(init["x_prev"], dtype=float)[keep].copy()
        w.g_prev = w.mat.T @ (w.mat @ w.x_prev + w.off)
    trace = []
    converged = False
    theta_out = np.zeros(m)
    gap_out = math.inf
    rounds = 0
    for rnd in range(round0 + 1, round0 + limit + 1):
        rounds = rnd
        optimal = False
        if kind == "pg":
            pg_passes(w, eta, inner_passes)
        elif kind == "apg":
            apg_passes(w, eta, inner_passes, mom, restart)
        elif kind == "cd":
            cd_passes(w, inner_passes)
        else:
            passive = passive_full[w.idx]
            optimal = active_set_pass(w, passive)
            passive_full[w.idx] = passive

        # dual point on the reduced problem (driver.py:183-201)
        theta = -w.r
        v = -w.g
        eps = 0.0
        if inf_mask.any():
            here = inf_mask[w.idx]
            att = att_full[w.idx]
            if here.any():
                eps = float(np.max(np.maximum(v[here], 0.0) / np.abs(att[here])))
            if eps > 0.0:
                theta = theta + eps * t
            v = v + eps * att
        primal = 0.5 * float(w.r @ w.r)
        dual = float(theta @ w.tgt) - 0.5 * float(theta @ theta)
        dual -= float(lo[w.idx] @ np.minimum(v, 0.0))
        fin = ~inf_mask[w.idx]
        if fin.any():
            dual -= float(hi[w.idx][fin] @ np.maximum(v[fin], 0.0))
        gap = clamp(primal - dual)
        theta_out, gap_out = theta, gap
        cert = None
        if gap < gap_tol:
            w.write_back(x_full)
            cert, th_c, _, _ = certified_gap(a, y, lo, hi, inf_mask, x_full, t, att_full)
            theta_out, gap_out = th_c, cert
            if cert < gap_tol:
                converged = True

        rec = dict(round=rnd, primal=primal, dual=dual, gap=gap, eps=eps,
                   step=eta, certified=cert)
        new_lo = new_up = np.empty(0, dtype=int)
        radius = slack = math.nan
        if screening:
            radius = math.sqrt(2.0 * gap / 1.0)
            slack = SLACK_SCALE * max(1.0, float(np.linalg.norm(theta)))
            thr = (radius + slack) * norms[w.idx]
            new_lo = w.idx[v < -thr]
            new_up = w.idx[(v > thr) & fin]
            if new_lo.size or new_up.size:
                w.write_back(x_full)
                x_full[new_lo] = lo[new_lo]
                x_full[new_up] = hi[new_up]
                if new_lo.size:
                    z += a[:, new_lo] @ lo[new_lo]
                if new_up.size:
                    z += a[:, new_up] @ hi[new_up]
                sat_lo = np.concatenate([sat_lo, new_lo])
                sat_up = np.concatenate([sat_up, new_up])
                gone = np.concatenate([new_lo, new_up])
                keep = keep[~np.isin(keep, gone)]
                if kind == "active-set":
                    passive_full[gone] = False   # ActiveSetState.drop_screened
                old = w
                w = ActiveView(a, y, lo, hi, norms, z, x_full, keep)
                if kind == "apg" and old.x_prev is not None:
                    xp_full = x_full.copy()
                    xp_full[old.idx] = old.x_prev
                    xp_full[gone] = x_full[gone]
                    w.x_prev = xp_full[keep].copy()
                    w.g_prev = w.mat.T @ (w.mat @ w.x_prev + w.off)
                if (kind in ("pg", "apg") and step_size is None
                        and keep.size < 0.5 * basis):
                    eta = safe_step(w.mat, 1.0, power_iters)
                    basis = keep.size
        rec.update(radius=radius, slack=slack, preserved=int(keep.size),
                   new_lower=int(new_lo.size), new_upper=int(new_up.size))
        if record_sets:
            rec.update(new_lower_idx=new_lo.copy(), new_upper_idx=new_up.copy())
        trace.append(rec)
        if round_hook is not None:
            round_hook(rnd, w, rec)
        if converged:
            break
        if optimal:
            # KKT-optimal active set: decided by the certified gap alone
            # (driver.py:246-252)
            w.write_back(x_full)
            cert, th_c, _, _ = certified_gap(a, y, lo, hi, inf_mask, x_full, t, att_full)
            theta_out, gap_out = th_c, cert
            converged = cert < gap_tol
            break
    w.write_back(x_full)
    return dict(x=x_full.copy(), theta=np.asarray(theta_out).copy(), gap=gap_out,
                rounds=rounds, converged=converged, trace=trace,
                sat_lower=sat_lo.copy(), sat_upper=sat_up.copy(), step=eta)


def objective(a, y, x):
    r = a @ x - y
    return 0.5 * float(r @ r)

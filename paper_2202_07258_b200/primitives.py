"""The reference's spec-level per-round primitives, on the GPU.

Drop-in for the per-round API /root/reference/pkg/src/boxscreen/__init__.py
exports next to ``solve``: the dual-point family (duality.py:103-209), the
screening bookkeeping (screening.py:18-104) and the one-shot primal updates
(solvers.py:207-227).  Same names, arguments, return values and exceptions;
host numpy in and out, like the reference.  Every O(m n) operation runs in the
native library through the fine-grained C ABI (include/boxscreen_b200.h:
bx_set_state, bx_primal_passes, bx_gradient, bx_apply_a, bx_apply_at,
bx_dual_point, bx_eval_dual, bx_sphere_test) on a device context cached on
the Problem; PyTorch only moves buffers and does O(n) index bookkeeping.
There is no CPU path: without CUDA / the library these raise.
"""

import ctypes
import math

import numpy as np

from . import _native as nat
from .errors import (DimensionMismatch, DualInfeasible, IndexOutOfPreserved, InternalConsistency,
                     NotInterior, WrongVariant, ZeroColumn)
from .model import PrimalPoint

FEASIBILITY_TOL = 1e-12  # duality.py:21
GAP_ROUNDOFF = 1e-9      # duality.py:24


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

def _session(p, t=None):
    from .driver import device_session
    return device_session(p, t)


def _dev(arr, s, dtype=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(arr, dtype=dtype or np.float64), device=s.dev["a"].device)


def _empty(s, n, dtype=None):
    import torch
    return torch.empty(max(int(n), 1), dtype=dtype or torch.float64, device=s.dev["a"].device)


def _host(t, n=None):
    a = t.cpu().numpy()
    return a if n is None else a[:n]


def _apply_at(s, v_dev):
    out = _empty(s, s.n)
    nat.check(nat.lib().bx_apply_at(s.ctx, v_dev.data_ptr(), out.data_ptr()), s.ctx, "bx_apply_at")
    return out[: s.n]


def _apply_a(s, coef_dev, cols_dev=None, z_add_dev=None):
    out = _empty(s, s.m)
    k = s.n if cols_dev is None else int(cols_dev.numel())
    nat.check(nat.lib().bx_apply_a(s.ctx, None if cols_dev is None else cols_dev.data_ptr(), k,
                                   coef_dev.data_ptr() if k else None,
                                   None if z_add_dev is None else z_add_dev.data_ptr(), out.data_ptr()),
              s.ctx, "bx_apply_a")
    return out[: s.m]


def _check_theta(p, theta):
    theta = np.asarray(theta, dtype=float).ravel()
    if theta.shape[0] != p.m:
        raise DimensionMismatch(f"theta has length {theta.shape[0]}, expected {p.m}")
    return theta


def device_col_norms(p):
    """||a_j||_2 from the GPU setup pass (model.py:89-92)."""
    import torch
    s = _session(p)
    out = torch.empty(p.n, dtype=torch.float64, device=s.dev["a"].device)
    nat.check(nat.lib().bx_col_norms(s.ctx, out.data_ptr()), s.ctx, "bx_col_norms")
    return out.cpu().numpy()


def device_forward(p, x):
    """A x on the GPU (model.py:117's a_matrix @ x)."""
    s = _session(p)
    return _host(_apply_a(s, _dev(x, s)))


# ---------------------------------------------------------------------------
# duality (duality.py:29-209)
# ---------------------------------------------------------------------------

class DualState:
    """Dual point, its objective, the gap and the cached A'theta (duality.py:29-38)."""

    __slots__ = ("theta", "d_value", "gap", "a_t_theta_cache")

    def __init__(self, theta, d_value, gap, a_t_theta_cache):
        self.theta = theta
        self.d_value = d_value
        self.gap = gap
        self.a_t_theta_cache = a_t_theta_cache


def eval_dual(p, theta, a_t_theta=None):
    """D(theta) = sum theta_i y_i - theta_i^2/2 - l'min(0, A'theta)
    - u_fin'max(0, A'theta) (duality.py:103-124); A'theta on the GPU when
    not given."""
    theta = _check_theta(p, theta)
    s = _session(p)
    th = _dev(theta, s)
    at = None if a_t_theta is None else _dev(np.asarray(a_t_theta, dtype=float).ravel(), s)
    d = ctypes.c_double()
    nat.check(nat.lib().bx_eval_dual(s.ctx, th.data_ptr(), None if at is None else at.data_ptr(), ctypes.byref(d)),
              s.ctx, "bx_eval_dual")
    return float(d.value)


def is_dual_feasible(p, theta, tol=FEASIBILITY_TOL):
    """a_j'theta <= tol for every infinite-upper column (duality.py:127-135)."""
    theta = _check_theta(p, theta)
    if p.j_inf.size == 0:
        return True
    s = _session(p)
    at = _apply_at(s, _dev(theta, s))
    jinf = _dev(p.j_inf, s, np.int64)
    return bool((at[jinf] <= tol).all())


def duality_gap(p, pt, theta):
    """P(x) - D(theta) for a feasible pair; raises below -1e-9 (duality.py:138-149)."""
    from .model import eval_primal
    if not is_dual_feasible(p, theta):
        raise DualInfeasible("theta is not dual feasible")
    gap = eval_primal(p, pt) - eval_dual(p, theta)
    if gap < -GAP_ROUNDOFF:
        raise InternalConsistency(f"duality gap {gap:.3e} below round-off slack")
    return gap


def _dual_point(p, pt, t):
    from .model import eval_primal
    eval_primal(p, pt)  # the box check (InfeasiblePoint), as the reference's gap evaluation does
    s = _session(p, t)
    x = _dev(pt.x, s)
    theta, at = _empty(s, s.m), _empty(s, s.n)
    out = (ctypes.c_double * 4)()
    nat.check(nat.lib().bx_dual_point(s.ctx, x.data_ptr(), 1.0, theta.data_ptr(), at.data_ptr(), out),
              s.ctx, "bx_dual_point")
    return DualState(_host(theta, s.m), float(out[2]), float(out[0]), _host(at, s.n))


def dual_point_bvlr(p, pt):
    """Dual scaling theta = y - A x (duality.py:159-168); every upper bound finite."""
    if p.j_inf.size:
        raise WrongVariant("dual scaling needs every upper bound finite")
    return _dual_point(p, pt, None)


def dual_point_nnlr(p, tv, pt):
    """Dual translation theta = Xi_t(y - A x) (duality.py:187-209)."""
    if np.any(np.asarray(tv.a_t_t) >= 0):
        raise NotInterior("translation vector is not strictly interior")
    return _dual_point(p, pt, tv.t)


def dual_translate(p, tv, z):
    """z + eps t with eps = max_j max(0, a_j'z) / |a_j't| (duality.py:171-184)."""
    z = np.asarray(z, dtype=float).ravel()
    if z.shape[0] != p.m:
        raise DimensionMismatch(f"z has length {z.shape[0]}, expected {p.m}")
    att = np.asarray(tv.a_t_t, dtype=float)
    if np.any(att >= 0):
        raise NotInterior("translation vector is not strictly interior")
    s = _session(p)
    atz = _apply_at(s, _dev(z, s))
    eps = float((atz.clamp(min=0.0) / _dev(np.abs(att), s)).max())
    return z + eps * np.asarray(tv.t, dtype=float)


# ---------------------------------------------------------------------------
# screening (screening.py:18-104)
# ---------------------------------------------------------------------------

class ScreeningState:
    """Preserved set, saturated sets, saturated part z, column norms, radius
    (screening.py:18-43); the norms come from the GPU setup pass."""

    def __init__(self, p):
        norms = device_col_norms(p)
        if np.any(norms == 0.0):
            raise ZeroColumn(f"zero column at index {int(np.argmin(norms))}")
        self.preserved = np.arange(p.n)
        self.sat_lower = np.empty(0, dtype=int)
        self.sat_upper = np.empty(0, dtype=int)
        self.z = np.zeros(p.m)
        self.col_norms = norms
        self.radius = math.inf

    @property
    def preserved_count(self):
        return int(self.preserved.size)

    def screening_ratio(self, n):
        return (n - self.preserved.size) / n


def safe_screen_test(st, a_t_theta, p, slack=0.0):
    """Strict sphere test on the preserved coordinates (screening.py:46-69):
    returns (new_lower, new_upper) original indices."""
    import torch
    a_t_theta = np.asarray(a_t_theta, dtype=float)
    if a_t_theta.shape[0] != p.n:
        raise DimensionMismatch("a_t_theta must have length n")
    idx = st.preserved
    if idx.size == 0:
        return np.empty(0, dtype=int), np.empty(0, dtype=int)
    s = _session(p)
    v = _dev(a_t_theta, s)
    pres = _dev(idx, s, np.int32)
    flags = torch.empty(idx.size, dtype=torch.uint8, device=v.device)
    nat.check(nat.lib().bx_sphere_test(s.ctx, v.data_ptr(), pres.data_ptr(), idx.size, float(st.radius),
                                       float(slack), flags.data_ptr()), s.ctx, "bx_sphere_test")
    f = flags.cpu().numpy()
    return idx[f == 1], idx[f == 2]


def apply_screening(st, new_lower, new_upper, pt, p):
    """Fix the newly screened coordinates at their bounds, fold them into z,
    shrink the preserved set (screening.py:72-94); z += A_S b_S on the GPU."""
    new_lower = np.asarray(new_lower, dtype=int)
    new_upper = np.asarray(new_upper, dtype=int)
    if new_lower.size == 0 and new_upper.size == 0:
        return st
    newly = np.concatenate([new_lower, new_upper])
    if not np.isin(newly, st.preserved).all():
        raise IndexOutOfPreserved("screened index not in the preserved set")
    pt.x[new_lower] = p.lower[new_lower]
    pt.x[new_upper] = p.upper[new_upper]
    s = _session(p)
    coef = np.concatenate([p.lower[new_lower], p.upper[new_upper]])
    st.z = _host(_apply_a(s, _dev(coef, s), _dev(newly, s, np.int32), _dev(st.z, s)))
    st.sat_lower = np.concatenate([st.sat_lower, new_lower])
    st.sat_upper = np.concatenate([st.sat_upper, new_upper])
    st.preserved = st.preserved[~np.isin(st.preserved, newly)]
    return st


def forward_product(st, p, x_preserved):
    """A[:, preserved] x_preserved + z (screening.py:97-104)."""
    x_preserved = np.asarray(x_preserved, dtype=float)
    if x_preserved.shape[0] != st.preserved.size:
        raise DimensionMismatch("x_preserved must match the preserved set size")
    if st.preserved.size == 0:
        return st.z.copy()
    s = _session(p)
    return _host(_apply_a(s, _dev(x_preserved, s), _dev(st.preserved, s, np.int32), _dev(st.z, s)))


# ---------------------------------------------------------------------------
# one-shot primal updates (solvers.py:207-227)
# ---------------------------------------------------------------------------

def _update(p, st, pt, kind, eta, passes):
    s = _session(p)
    L = nat.lib()
    pres = np.ascontiguousarray(st.preserved, dtype=np.int64)
    x = _dev(pt.x, s)
    z = _dev(st.z, s)
    nat.check(L.bx_set_state(s.ctx, pres.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pres.size, x.data_ptr(),
                             z.data_ptr()), s.ctx, "bx_set_state")
    nat.check(L.bx_primal_passes(s.ctx, nat.KINDS[kind], float(eta), int(passes)), s.ctx, "bx_primal_passes")
    resid, grad = _empty(s, s.m), _empty(s, pres.size)
    nat.check(L.bx_gradient(s.ctx, resid.data_ptr(), grad.data_ptr()), s.ctx, "bx_gradient")
    xo = _empty(s, s.n)
    nat.check(L.bx_get_state(s.ctx, xo.data_ptr(), None, None, None), s.ctx, "bx_get_state")
    r = _host(resid, s.m)
    pt.x = _host(xo, s.n).copy()
    pt.ax_cache = r + p_y(p)
    return r, _host(grad, pres.size)


def p_y(p):
    return p.y if p.y is not None else p.device_arrays()["y"].cpu().numpy()


class ActiveSetState:
    """Passive (free) set of the active-set solver (solvers.py:38-45)."""

    def __init__(self, n):
        self.passive = np.zeros(n, dtype=bool)

    def drop_screened(self, preserved_mask):
        self.passive &= preserved_mask


def active_set_update(p, st, pt, as_state, cfg):
    """One outer bounded-variable Lawson-Hanson iteration on the preserved
    set; returns (residual, restricted gradient, optimal) and updates pt and
    as_state.passive (solvers.py:229-240)."""
    import torch
    s = _session(p)
    if getattr(s, "as_ws", None) is None:
        s.attach_active_set()
    L = nat.lib()
    pres = np.ascontiguousarray(st.preserved, dtype=np.int64)
    x = _dev(pt.x, s)
    z = _dev(st.z, s)
    nat.check(L.bx_set_state(s.ctx, pres.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pres.size, x.data_ptr(),
                             z.data_ptr()), s.ctx, "bx_set_state")
    pin = torch.as_tensor(as_state.passive[pres].astype(np.uint8), device=x.device)
    pout = torch.empty(max(pres.size, 1), dtype=torch.uint8, device=x.device)
    opt = ctypes.c_int32()
    nat.check(L.bx_active_set_step(s.ctx, pin.data_ptr(), pout.data_ptr(), ctypes.byref(opt)), s.ctx,
              "bx_active_set_step")
    as_state.passive[pres] = pout.cpu().numpy()[: pres.size].astype(bool)
    resid, grad = _empty(s, s.m), _empty(s, pres.size)
    nat.check(L.bx_gradient(s.ctx, resid.data_ptr(), grad.data_ptr()), s.ctx, "bx_gradient")
    xo = _empty(s, s.n)
    nat.check(L.bx_get_state(s.ctx, xo.data_ptr(), None, None, None), s.ctx, "bx_get_state")
    r = _host(resid, s.m)
    pt.x = _host(xo, s.n).copy()
    pt.ax_cache = r + p_y(p)
    return r, _host(grad, pres.size), bool(opt.value)


def pg_update(p, st, pt, cfg, step_size):
    """cfg.inner_passes projected-gradient passes on the preserved set; returns
    (residual, restricted gradient) and updates pt (solvers.py:207-217)."""
    return _update(p, st, pt, "pg", step_size, cfg.inner_passes)


def cd_update(p, st, pt, cfg):
    """cfg.inner_passes cyclic coordinate-descent sweeps (solvers.py:220-226)."""
    return _update(p, st, pt, "cd", 1.0, cfg.inner_passes)


__all__ = ["ActiveSetState", "active_set_update", "DualState", "ScreeningState", "apply_screening", "cd_update", "device_col_norms", "device_forward",
           "dual_point_bvlr", "dual_point_nnlr", "dual_translate", "duality_gap", "eval_dual", "forward_product",
           "is_dual_feasible", "pg_update", "safe_screen_test", "PrimalPoint"]

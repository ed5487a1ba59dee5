"""Problem container and the quadratic loss (reference: model.py:8-120).

``Problem`` validates exactly as the reference does (model.py:55-87) and keeps
host arrays; it also accepts CUDA tensors (already resident in HBM), in which
case nothing is copied through the host.  ``dtype`` selects fp64 (reference
behaviour, model.py:56) or fp32 storage (BASELINE config 4).  Device copies
are column-major with a 16-byte-aligned column stride, as the C ABI requires.
"""

import numpy as np

from .errors import DimensionMismatch, InfeasiblePoint


def eval_loss(z, y):
    """0.5 (z - y)^2 (model.py:8-11)."""
    d = np.asarray(z, dtype=float) - np.asarray(y, dtype=float)
    return 0.5 * d * d if d.ndim else 0.5 * float(d) ** 2


def grad_loss(z, y):
    """z - y (model.py:14-17)."""
    d = np.asarray(z, dtype=float) - np.asarray(y, dtype=float)
    return d if d.ndim else float(d)


def conj_loss(u, y):
    """u y + 0.5 u^2 (model.py:20-29)."""
    u = np.asarray(u, dtype=float)
    y = np.asarray(y, dtype=float)
    v = u * y + 0.5 * u * u
    return v if v.ndim else float(v)


class QuadraticLoss:
    """model.py:32-44; alpha = 1 is the dual's strong-concavity constant."""

    alpha = 1.0
    value = staticmethod(eval_loss)
    grad = staticmethod(grad_loss)
    conjugate = staticmethod(conj_loss)


def _readonly_view(arr):
    """Zero-copy torch view of a (read-only, like the reference's Problem
    arrays, model.py:85-87) C-contiguous numpy array; it is only ever read."""
    import warnings

    import torch
    arr = np.ascontiguousarray(arr)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def _is_torch(x):
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _validate_device(a, y, lo, hi):
    """The reference's input checks (model.py:58-76) on CUDA tensors, in the
    same order and with the same messages as the host path; each check is a
    device reduction, only its boolean comes back."""
    import torch
    if bool(torch.isnan(a).any()) or bool(torch.isnan(y).any()):
        raise ValueError("NaN entries in A or y")
    if bool(torch.isnan(lo).any()) or bool(torch.isnan(hi).any()):
        raise ValueError("NaN entries in bounds")
    if not bool(torch.isfinite(lo).all()):
        raise ValueError("lower bounds must be finite")
    if bool(torch.isinf(a).any()) or bool(torch.isinf(y).any()):
        raise ValueError("A and y must be finite")
    if not bool((lo < hi).all()):
        raise ValueError("need lower_j < upper_j for every coordinate")


class Problem:
    """min 0.5 ||A x - y||^2  s.t.  lower <= x <= upper  (model.py:47-99)."""

    def __init__(self, a_matrix, y, lower, upper, dtype=None, pin=False):
        if _is_torch(a_matrix) and a_matrix.is_cuda:
            self._init_device(a_matrix, y, lower, upper, dtype)
            return
        np_dtype = np.dtype(dtype) if dtype is not None else np.dtype(np.float64)
        if np_dtype not in (np.float64, np.float32):
            raise ValueError("dtype must be float64 or float32")
        a = np.array(a_matrix, dtype=np_dtype, order="F")
        y = np.array(y, dtype=float).ravel()
        if a.ndim != 2:
            raise DimensionMismatch("A must be a 2-d matrix")
        m, n = a.shape
        if m < 1 or n < 1:
            raise DimensionMismatch("A must have at least one row and column")
        if y.shape[0] != m:
            raise DimensionMismatch(f"y has length {y.shape[0]}, expected {m}")
        lower = np.broadcast_to(np.asarray(lower, dtype=float), (n,)).copy()
        upper = np.broadcast_to(np.asarray(upper, dtype=float), (n,)).copy()
        if np.isnan(a).any() or np.isnan(y).any():
            raise ValueError("NaN entries in A or y")
        if np.isnan(lower).any() or np.isnan(upper).any():
            raise ValueError("NaN entries in bounds")
        if not np.all(np.isfinite(lower)):
            raise ValueError("lower bounds must be finite")
        if np.isinf(a).any() or np.isinf(y).any():
            raise ValueError("A and y must be finite")
        if not np.all(lower < upper):
            raise ValueError("need lower_j < upper_j for every coordinate")
        self.dtype = np_dtype
        self.a_matrix = a
        self.y = y
        self.lower = lower
        self.upper = upper
        self.m = m
        self.n = n
        self.j_inf_mask = np.isinf(upper)
        self.j_inf = np.flatnonzero(self.j_inf_mask)
        for arr in (self.a_matrix, self.y, self.lower, self.upper, self.j_inf_mask, self.j_inf):
            arr.setflags(write=False)
        self._dev = None
        self._pinned = None
        if pin:
            self.pin()

    def _init_device(self, a, y, lower, upper, dtype):
        import torch
        m, n = a.shape
        tdt = a.dtype if dtype is None else (torch.float32 if np.dtype(dtype) == np.float32 else torch.float64)
        self.dtype = np.dtype(np.float32) if tdt == torch.float32 else np.dtype(np.float64)
        self.m, self.n = int(m), int(n)
        dev = a.device
        f64 = torch.float64  # every vector is fp64; only A has the storage dtype
        lo = torch.as_tensor(lower, dtype=f64, device=dev).broadcast_to((n,)).contiguous()
        hi = torch.as_tensor(upper, dtype=f64, device=dev).broadcast_to((n,)).contiguous()
        yv = torch.as_tensor(y, device=dev).to(f64).reshape(-1).contiguous()
        if yv.shape[0] != m:
            raise DimensionMismatch(f"y has length {yv.shape[0]}, expected {m}")
        _validate_device(a, yv, lo, hi)
        self._dev = dict(a=self._device_layout(a.to(tdt)), y=yv, lo=lo, hi=hi, device=dev)
        self.a_matrix = None
        self.y = None
        self.lower = lo.double().cpu().numpy()
        self.upper = hi.double().cpu().numpy()
        self.j_inf_mask = np.isinf(self.upper)
        self.j_inf = np.flatnonzero(self.j_inf_mask)
        self._pinned = None

    @classmethod
    def from_device_storage(cls, storage, m, y, lower, upper):
        """Wrap CUDA storage that already has the C-ABI layout: ``storage`` is
        (n, lda) row-major == column-major A with leading dimension lda >= m
        (e.g. a column block ``full_storage[c0:c1]`` of a larger problem)."""
        import torch
        p = cls.__new__(cls)
        n = storage.shape[0]
        tdt = storage.dtype
        p.dtype = np.dtype(np.float32) if tdt == torch.float32 else np.dtype(np.float64)
        p.m, p.n = int(m), int(n)
        dev = storage.device
        f64 = torch.float64
        lo = torch.as_tensor(lower, dtype=f64, device=dev).broadcast_to((n,)).contiguous()
        hi = torch.as_tensor(upper, dtype=f64, device=dev).broadcast_to((n,)).contiguous()
        yv = torch.as_tensor(y, device=dev).to(f64).reshape(-1).contiguous()
        if yv.shape[0] != m:
            raise DimensionMismatch(f"y has length {yv.shape[0]}, expected {m}")
        _validate_device(storage[:, :m], yv, lo, hi)
        p._dev = dict(a=storage, y=yv, lo=lo, hi=hi, device=dev)
        p.a_matrix = None
        p.y = None
        p.lower = lo.double().cpu().numpy()
        p.upper = hi.double().cpu().numpy()
        p.j_inf_mask = np.isinf(p.upper)
        p.j_inf = np.flatnonzero(p.j_inf_mask)
        p._pinned = None
        return p

    @staticmethod
    def _device_layout(a):
        """(m, n) tensor -> (n, lda) row-major storage == column-major A with a
        16-byte-aligned column stride."""
        import torch
        m, n = a.shape
        vec = 16 // a.element_size()
        lda = (m + vec - 1) // vec * vec
        if a.t().is_contiguous() and lda == m:
            return a.t()
        buf = torch.zeros((n, lda), dtype=a.dtype, device=a.device)
        buf[:, :m].copy_(a.t())
        return buf

    def pin(self):
        """Keep page-locked host copies so uploads run at full PCIe speed."""
        import torch
        if self._pinned is None and self.a_matrix is not None:
            at = _readonly_view(self.a_matrix.T)  # (n, m) == column-major A
            self._pinned = dict(a=at.pin_memory(), y=torch.from_numpy(self.y.copy()).pin_memory(),
                                lo=torch.from_numpy(self.lower.copy()).pin_memory(),
                                hi=torch.from_numpy(self.upper.copy()).pin_memory())
        return self

    def device_arrays(self, device=None):
        """Upload (once) and return the device copies {a (n, lda), y, lo, hi}."""
        import torch
        if self._dev is not None:
            return self._dev
        device = torch.device(device or "cuda")
        tdt = torch.float32 if self.dtype == np.float32 else torch.float64
        if self._pinned is not None:
            src = self._pinned
        else:
            src = dict(a=_readonly_view(self.a_matrix.T), y=torch.from_numpy(self.y.copy()),
                       lo=torch.from_numpy(self.lower.copy()), hi=torch.from_numpy(self.upper.copy()))
        nb = self._pinned is not None
        at = src["a"].to(device, non_blocking=nb)
        a_dev = self._device_layout(at.t()) if at.shape[1] % (16 // at.element_size()) else at
        self._dev = dict(a=a_dev, y=src["y"].to(device, non_blocking=nb),
                         lo=src["lo"].to(device, non_blocking=nb),
                         hi=src["hi"].to(device, non_blocking=nb), device=device)
        return self._dev

    def release_device(self):
        """Drop the cached device copies (the next solve uploads again)."""
        self._dev = None

    @property
    def col_norms(self):
        """||a_j||_2 (model.py:89-92), from the GPU setup pass."""
        from .primitives import device_col_norms
        return device_col_norms(self)

    def is_box_feasible(self, x):
        x = np.asarray(x, dtype=float)
        if x.shape != (self.n,):
            raise DimensionMismatch(f"x has shape {x.shape}, expected ({self.n},)")
        return bool(np.all(x >= self.lower) and np.all(x <= self.upper))


class PrimalPoint:
    """Box-feasible primal candidate with an optional cached forward product (model.py:101-106)."""

    def __init__(self, x, ax_cache=None):
        self.x = np.array(x, dtype=float).ravel()
        self.ax_cache = None if ax_cache is None else np.array(ax_cache, dtype=float).ravel()


def eval_primal(p, pt):
    """0.5 ||A x - y||^2 with an exact box check (model.py:109-120)."""
    if not p.is_box_feasible(pt.x):
        raise InfeasiblePoint("primal point violates the box constraint")
    if pt.ax_cache is not None:
        ax = pt.ax_cache
    else:
        from .primitives import device_forward  # A x on the GPU (bx_apply_a)
        ax = device_forward(p, pt.x)
    if ax.shape != (p.m,):
        raise DimensionMismatch("ax_cache has wrong length")
    y = p.y if p.y is not None else p.device_arrays()["y"].cpu().numpy()
    r = ax - y
    return 0.5 * float(r @ r)

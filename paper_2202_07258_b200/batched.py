"""Batched many-right-hand-side NNLS (BASELINE config 5): K problems sharing
one dictionary A, solved together by FISTA with per-problem Gap-safe
screening; both products of every step run on fp64 tensor cores (DMMA) inside
one persistent kernel per round (csrc/bx_batched.cuh).  Semantics:
oracle/batched_oracle.py ("Batched FISTA").  Not in the reference,
which solves one right-hand side per ``solve`` call."""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import STATUS, NativeError
from .solvers import auto_step_size


@dataclass
class BatchedResult:
    x: object                 # (n, K) numpy or CUDA tensor
    primal: np.ndarray        # per problem, last round
    dual: np.ndarray
    gap: np.ndarray
    eps: np.ndarray
    preserved: np.ndarray
    rounds: int
    converged: int
    iterations: int
    eta: float
    trace: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))  # per round: converged, max/mean gap, mean preserved
    kernel_launches: int = 0
    sphere_sweeps: int = 0    # tile-rounds that ran the per-coordinate sphere test (others cleared by the bound)
    tiles: int = 0            # tiles (64 right-hand sides) per round
    round_kernel_ms: float = 0.0   # summed duration of the round kernels (CUDA events)


def _check(st, h, what):
    if st != 0:
        msg = nat.lib().bx_batched_last_error(h)
        raise STATUS.get(st, NativeError)(f"{what}: {msg.decode() if msg else ''}")


def solve_batched(a, Y, passes=10, rounds=10, gap_tol=1e-6, screening=True, eta=None, return_device=False,
                  x_out=None, check_every=1):
    """Run up to ``rounds`` rounds of ``passes`` FISTA steps on every column of
    Y (m x K); stops early when every problem's gap < gap_tol.

    ``check_every``: rounds between convergence checks (1..16).  With more
    than one the device runs that many rounds per launch without a host round
    trip and overlaps the rounds of different tiles (the last, partly filled
    wave of a round runs beside the next round's first tiles); a batch that
    converges at an inner round still finishes its batch.

    ``x_out``: optional pinned host tensor (K x n, fp64) that receives X
    (returned as its n x K numpy view); reusing one across calls keeps the
    multi-GB device-to-host copy at full PCIe rate without a fresh pinned
    allocation per call."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2202_07258_b200 needs a CUDA device (no CPU fallback)")
    L = nat.lib()
    dev = torch.device("cuda")
    a_t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a, dtype=np.float64))
    y_t = Y if isinstance(Y, torch.Tensor) else torch.from_numpy(np.asarray(Y, dtype=np.float64))
    m, n = a_t.shape
    K = y_t.shape[1]
    lda = m + (m % 2)
    a_dev = torch.zeros((n, lda), dtype=torch.float64, device=dev)
    a_dev[:, :m].copy_(a_t.t().to(dev))
    y_dev = y_t.t().contiguous().to(dev, torch.float64)   # (K, m) == column-major Y, ldy = m
    if eta is None:
        eta = auto_step_size(a_dev[:, :m].t(), 1.0)
    nbytes = L.bx_batched_workspace_bytes(m, n, K)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    h = ctypes.c_void_p()
    try:
        _check(L.bx_batched_create(ctypes.byref(h), m, n, K, a_dev.data_ptr(), lda, y_dev.data_ptr(), m,
                                   ws.data_ptr(), nbytes, stream.cuda_stream), h, "bx_batched_create")
        if check_every != 1:
            _check(L.bx_batched_set_check_every(h, int(check_every)), h, "bx_batched_set_check_every")
        trace = np.zeros((rounds, 4))
        out = nat.BatchedOut()
        tr_p = trace.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        stats = torch.empty((5, K), dtype=torch.float64, device=dev)
        if return_device:
            _check(L.bx_batched_run(h, float(eta), passes, rounds, 1 if screening else 0, gap_tol, tr_p, rounds,
                                    ctypes.byref(out)), h, "bx_batched_run")
            x = torch.empty((K, n), dtype=torch.float64, device=dev)  # column-major n x K
            _check(L.bx_batched_get(h, x.data_ptr(), n, stats.data_ptr()), h, "bx_batched_get")
            xo = x.t()
        else:
            # n x K fp64 is GBs at config 5: the result goes to pinned host
            # memory (torch's caching host allocator reuses it across calls),
            # and the last round of the budget streams it out wave by wave
            # behind the remaining tensor work (bx_batched_run_to_host)
            host = x_out if x_out is not None else torch.empty((K, n), dtype=torch.float64, pin_memory=True)
            if tuple(host.shape) != (K, n) or host.dtype != torch.float64 or host.device.type != "cpu" or \
                    not host.is_contiguous():
                raise ValueError("x_out must be a contiguous (K, n) float64 host tensor")
            if not host.is_pinned():
                raise ValueError("x_out must be pinned host memory (torch.empty(..., pin_memory=True))")
            _check(L.bx_batched_run_to_host(h, float(eta), passes, rounds, 1 if screening else 0, gap_tol, tr_p, rounds,
                                            ctypes.byref(out), host.data_ptr(), n), h, "bx_batched_run_to_host")
            _check(L.bx_batched_get(h, None, n, stats.data_ptr()), h, "bx_batched_get")
            xo = host.numpy().T
    finally:
        L.bx_batched_destroy(h)
    st = stats.cpu().numpy()
    return BatchedResult(x=xo, primal=st[0], dual=st[1], gap=st[2], eps=st[3], preserved=st[4].astype(np.int64),
                         rounds=int(out.rounds), converged=int(out.converged), iterations=int(out.iterations),
                         eta=float(eta), trace=trace[: int(out.rounds)], kernel_launches=int(out.kernel_launches),
                         sphere_sweeps=int(out.sphere_sweeps), tiles=int(out.tiles),
                         round_kernel_ms=float(out.round_kernel_ms))

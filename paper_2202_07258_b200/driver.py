"""The screening solver front end: ``solve`` / ``SolveResult`` / ``TraceRecord``.

Drop-in for /root/reference/pkg/src/boxscreen/driver.py:131-256 (same
signature, same result and trace fields, same exceptions).  The whole
Algorithm-1 loop -- primal passes, dual point, gap, certified gap, sphere test,
compaction, step re-estimate -- runs natively in ``bx_solve``
(csrc/bx_core.cu) on one CUDA stream; this module owns the device buffers
(PyTorch) and converts results.  There is no CPU path: a missing native
library or a machine without CUDA raises.
"""

import csv
import ctypes
import json
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _native as nat
from .model import Problem, QuadraticLoss
from .solvers import SolverConfig, start_vector


@dataclass
class TraceRecord:
    round: int
    elapsed: float
    primal: float
    dual: float
    gap: float
    preserved_count: int
    screening_ratio: float
    newly_screened_lower: int = 0
    newly_screened_upper: int = 0


@dataclass
class SolveResult:
    x: np.ndarray
    theta: np.ndarray
    gap: float
    rounds: int
    converged: bool
    trace: list = field(default_factory=list)
    sat_lower: np.ndarray = field(default_factory=lambda: np.empty(0, int))
    sat_upper: np.ndarray = field(default_factory=lambda: np.empty(0, int))
    info: dict = field(default_factory=dict)

    def to_dict(self):
        d = asdict(self)
        d.pop("info", None)
        d["x"] = self.x.tolist()
        d["theta"] = self.theta.tolist()
        d["sat_lower"] = self.sat_lower.tolist()
        d["sat_upper"] = self.sat_upper.tolist()
        return d

    def to_json(self, path=None, indent=None):
        text = json.dumps(self.to_dict(), indent=indent)
        if path is not None:
            with open(path, "w") as fh:
                fh.write(text)
        return text


TRACE_CSV_COLUMNS = ("round", "elapsed_s", "primal", "dual", "gap", "preserved", "ratio")


def trace_to_csv(trace, path):
    """Byte-compatible with driver.py:72-80."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(TRACE_CSV_COLUMNS)
        for rec in trace:
            writer.writerow([rec.round, f"{rec.elapsed:.9f}", f"{rec.primal:.17g}", f"{rec.dual:.17g}",
                             f"{rec.gap:.17g}", rec.preserved_count, f"{rec.screening_ratio:.17g}"])


TRACE_DTYPE = np.dtype([("round", "<i8"), ("elapsed", "<f8"), ("primal", "<f8"), ("dual", "<f8"), ("gap", "<f8"),
                        ("preserved_count", "<i8"), ("newly_screened_lower", "<i8"),
                        ("newly_screened_upper", "<i8"), ("eps", "<f8"), ("radius", "<f8"), ("step", "<f8"),
                        ("certified_gap", "<f8"), ("restarts", "<i8"), ("momentum", "<f8")])
assert TRACE_DTYPE.itemsize == ctypes.sizeof(nat.TraceRec)


@ctypes.CFUNCTYPE(None, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p)
def _start_cb(k, seed, out, user):
    v = start_vector(int(k), int(seed))
    ctypes.memmove(out, v.ctypes.data, v.nbytes)


class _Session:
    """One native context over a Problem's device arrays (context manager)."""

    def __init__(self, p, tv=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2202_07258_b200 needs a CUDA device (no CPU fallback)")
        L = nat.lib()
        self.p = p
        d = p.device_arrays()
        self.dev = d
        self.torch = torch
        self.tdt = d["a"].dtype
        self.dtype_code = nat.BX_F32 if self.tdt == torch.float32 else nat.BX_F64
        a = d["a"]  # (n, lda) storage of column-major A
        self.m, self.n = p.m, p.n
        lda = a.stride(0)
        nbytes = L.bx_workspace_bytes(self.m, self.n, self.dtype_code)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=a.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(a.device)
        self.t_dev = None
        if tv is not None:
            self.t_dev = torch.as_tensor(np.asarray(tv.t, dtype=np.float64), device=a.device).contiguous()
        if stream is not None:
            # the device arrays (upload / layout copy) and t were produced on
            # the current stream: order the context's first kernels after them
            stream.wait_stream(torch.cuda.current_stream(a.device))
        self.ctx = ctypes.c_void_p()
        st = L.bx_ctx_create(ctypes.byref(self.ctx), self.m, self.n, self.dtype_code, a.data_ptr(), lda,
                             d["y"].data_ptr(), d["lo"].data_ptr(), d["hi"].data_ptr(),
                             self.t_dev.data_ptr() if self.t_dev is not None else None,
                             self.ws.data_ptr(), nbytes, self.stream.cuda_stream)
        if st != 0:
            try:
                nat.check(st, self.ctx, "bx_ctx_create")
            finally:
                L.bx_ctx_destroy(self.ctx)
                self.ctx = None

    def attach_group(self, group, rank, col_offset, n_global):
        nat.check(nat.lib().bx_ctx_set_group(self.ctx, group, rank, col_offset, n_global), self.ctx,
                  "bx_ctx_set_group")

    def attach_nccl(self, uid, rank, nranks, col_offset, n_global):
        nat.check(nat.lib().bx_ctx_set_comm(self.ctx, uid, rank, nranks, col_offset, n_global), self.ctx,
                  "bx_ctx_set_comm")

    def use_comm(self, comm, col_offset, n_global):
        """Borrow a persistent communicator (distributed.ShardComm)."""
        nat.check(nat.lib().bx_ctx_use_comm(self.ctx, comm.handle, col_offset, n_global), self.ctx,
                  "bx_ctx_use_comm")

    def attach_peers(self, gather=None, agree=None):
        """Fused reduce + peer exchange for the per-step reduction
        (csrc/bx_exchange.cuh).  ``gather(handle_bytes) -> list of every
        rank's handle`` for NCCL ranks (one GPU each); None for the
        in-process group.  ``agree(ok) -> bool`` is True when every rank
        mapped its peers (an all-reduce over the ranks)."""
        L = nat.lib()
        if gather is None:
            nat.check(L.bx_peer_alloc(self.ctx, None), self.ctx, "bx_peer_alloc")
            nat.check(L.bx_peer_open(self.ctx, None), self.ctx, "bx_peer_open")
            return
        # every rank takes part in the gather and the agreement even when its
        # own step failed, so no rank is left waiting in a collective; if
        # any rank cannot map its peers, all fall back to the NCCL schedule
        h = ctypes.create_string_buffer(64)
        ok = L.bx_peer_alloc(self.ctx, h) == 0
        handles = b"".join(gather(h.raw))
        ok = ok and L.bx_peer_open(self.ctx, handles) == 0
        if agree is not None and not agree(ok):
            nat.check(L.bx_peer_disable(self.ctx), self.ctx, "bx_peer_disable")
            import warnings
            warnings.warn("fused peer exchange unavailable on some rank; using the NCCL schedule")
        elif not ok:
            nat.check(L.bx_peer_open(self.ctx, handles), self.ctx, "bx_peer_open")  # raise with the message

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def close(self):
        if self.ctx is not None:
            nat.lib().bx_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def power_iter(self, iters, v0):
        nat.check(nat.lib().bx_reset(self.ctx), self.ctx, "bx_reset")
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        sig = ctypes.c_double()
        nat.check(nat.lib().bx_power_iter(self.ctx, iters, v0.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                          ctypes.byref(sig)), self.ctx, "bx_power_iter")
        return sig.value

    def attach_active_set(self):
        """Scratch of the active-set kind: the passive Cholesky factor
        (min(m, n)^2 fp64) and its vectors, owned here like the workspace."""
        L = nat.lib()
        nbytes = L.bx_active_set_workspace_bytes(self.m, self.n)
        self.as_ws = self.torch.empty(nbytes, dtype=self.torch.uint8, device=self.ws.device)
        nat.check(L.bx_ctx_set_active_set_workspace(self.ctx, self.as_ws.data_ptr(), nbytes), self.ctx,
                  "bx_ctx_set_active_set_workspace")

    def run(self, cfg, screening, alpha, slack_scale, profile=False, prev_iterate=False):
        L = nat.lib()
        if cfg.kind == "active-set" and getattr(self, "as_ws", None) is None:
            self.attach_active_set()
        nat.check(L.bx_set_profiling(self.ctx, 1 if profile else 0), self.ctx, "bx_set_profiling")
        c = nat.SolveCfg()
        c.kind = nat.KINDS[cfg.kind]
        c.inner_passes = cfg.inner_passes
        c.max_rounds = cfg.max_rounds or 0
        c.gap_tol = cfg.gap_tol
        c.step_size = cfg.step_size if cfg.step_size is not None else float("nan")
        c.power_iters = cfg.power_iters
        c.screening = 1 if screening else 0
        c.alpha = alpha
        c.slack_scale = slack_scale
        rel = cfg.relative_gap
        c.relative_gap = int(self.dtype_code == nat.BX_F32 if rel is None else bool(rel))
        c.restart = nat.RESTARTS[cfg.restart]
        cap = min(cfg.max_rounds or 1_000_000, 250_000)
        trace = np.empty(cap, dtype=TRACE_DTYPE)
        out = nat.SolveOut()
        st = L.bx_solve(self.ctx, ctypes.byref(c), _start_cb, None,
                        trace.ctypes.data_as(ctypes.POINTER(nat.TraceRec)), cap, ctypes.byref(out))
        nat.check(st, self.ctx, "bx_solve")
        self.profile = None
        if profile:
            ents = (nat.ProfEntry * nat.PROF_SLOTS)()
            nat.check(L.bx_get_profile(self.ctx, ents, nat.PROF_SLOTS), self.ctx, "bx_get_profile")
            self.profile = {nat.PROF_NAMES[i]: dict(launches=int(e.launches), ms=float(e.ms), bytes=float(e.bytes))
                            for i, e in enumerate(ents) if e.launches}
        torch = self.torch
        dev = self.dev["a"].device
        x = torch.empty(self.n, dtype=torch.float64, device=dev)
        theta = torch.empty(self.m, dtype=torch.float64, device=dev)
        sl = torch.empty(max(out.n_sat_lower, 1), dtype=torch.int64, device=dev)
        su = torch.empty(max(out.n_sat_upper, 1), dtype=torch.int64, device=dev)
        nat.check(L.bx_get_state(self.ctx, x.data_ptr(), theta.data_ptr(), sl.data_ptr(), su.data_ptr()),
                  self.ctx, "bx_get_state")
        self.x_prev = None
        if prev_iterate:
            xp = torch.empty(self.n, dtype=torch.float64, device=dev)
            nat.check(L.bx_get_prev_iterate(self.ctx, xp.data_ptr()), self.ctx, "bx_get_prev_iterate")
            self.x_prev = xp.cpu().numpy()
        return out, trace[: min(out.rounds, cap)], x, theta, sl[: out.n_sat_lower], su[: out.n_sat_upper]


def device_session(p, t=None):
    """A native context over ``p`` (and translation vector ``t``), created
    once and cached on the Problem: the spec-level primitives
    (primitives.py) run their passes on it."""
    import types
    key = None if t is None else np.asarray(t, dtype=np.float64).ravel().tobytes()
    cache = p.__dict__.setdefault("_sessions", {})
    s = cache.get(key)
    if s is None or s.ctx is None:
        tv = None if t is None else types.SimpleNamespace(t=np.asarray(t, dtype=np.float64).ravel())
        s = _Session(p, tv=tv)
        cache[key] = s
    return s


def column_stats(p, t=None):
    """(||a_j||, A't) computed on the GPU (k_colstats, the setup pass of
    bx_ctx_create) as host fp64 arrays; A't is None without ``t``."""
    import types
    tv = None if t is None else types.SimpleNamespace(t=np.asarray(t, dtype=np.float64).ravel())
    with _Session(p, tv=tv) as s:
        torch = s.torch
        dev = s.dev["a"].device
        nrm = torch.empty(p.n, dtype=torch.float64, device=dev)
        nat.check(nat.lib().bx_col_norms(s.ctx, nrm.data_ptr()), s.ctx, "bx_col_norms")
        att = None
        if tv is not None:
            att_d = torch.empty(p.n, dtype=torch.float64, device=dev)
            nat.check(nat.lib().bx_att(s.ctx, att_d.data_ptr()), s.ctx, "bx_att")
            att = att_d.cpu().numpy()
        return nrm.cpu().numpy(), att


def _result(p_n, out, tr, x, theta, sl, su, prof, return_device, n_total=None):
    n = n_total or p_n
    trace = [TraceRecord(int(r["round"]), float(r["elapsed"]), float(r["primal"]), float(r["dual"]),
                         float(r["gap"]), int(r["preserved_count"]), (n - int(r["preserved_count"])) / n,
                         int(r["newly_screened_lower"]), int(r["newly_screened_upper"])) for r in tr]
    info = dict(iterations=int(out.iterations), step=float(out.step), sigma=float(out.sigma),
                kernel_launches=int(out.kernel_launches), restarts=int(out.restarts), trace_arrays=tr, profile=prof,
                spec_kept=int(out.spec_kept), spec_undone=int(out.spec_undone))
    if return_device:
        xo, tho = x, theta
    else:
        xo = x.double().cpu().numpy()
        tho = theta.double().cpu().numpy()
    return SolveResult(x=xo, theta=tho, gap=float(out.gap), rounds=int(out.rounds), converged=bool(out.converged),
                       trace=trace, sat_lower=sl.cpu().numpy(), sat_upper=su.cpu().numpy(), info=info)


def _default_slack(p):
    # driver.py:219 for fp64; fp32 sphere tests need a slack above the fp32
    # round-off of a_j'theta (~sqrt(m) * 6e-8 ||theta||): 1e-4 ||theta||
    return 1e-12 if p.dtype == np.float64 else 1e-4


def solve(p, cfg=None, screening=True, tv=None, loss=QuadraticLoss, slack_scale=None, return_device=False,
          profile=False, prev_iterate=False):
    """Run the chosen primal solver with (or without) dynamic safe screening.

    Same contract as the reference's ``solve`` (driver.py:131-256).  With
    ``return_device`` the result's x / theta stay CUDA tensors (no host copy);
    ``profile`` times every kernel launch with CUDA events (info["profile"]);
    ``prev_iterate`` adds FISTA's previous iterate (info["x_prev"]), which with
    the last trace record's momentum is the state a round resumes from.
    """
    cfg = cfg or SolverConfig()
    if not isinstance(p, Problem):
        raise TypeError("p must be a Problem")
    if slack_scale is None:
        slack_scale = _default_slack(p)
    with _Session(p, tv=tv) as s:
        out, tr, x, theta, sl, su = s.run(cfg, screening, loss.alpha, slack_scale, profile=profile,
                                          prev_iterate=prev_iterate)
        prof = s.profile
        x_prev = s.x_prev
    res = _result(p.n, out, tr, x, theta, sl, su, prof, return_device)
    if prev_iterate:
        res.info["x_prev"] = x_prev
    return res

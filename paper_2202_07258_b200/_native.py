"""ctypes binding of the C ABI in include/boxscreen_b200.h.

The shared library ``_lib/libboxscreen_b200.so`` is built in-tree by
``paper_2202_07258_b200.build`` (nvcc, sm_100a).  There is no CPU fallback:
importing this module raises when the library is missing, and every call
that fails raises the reference exception class its status code maps to.
"""

import ctypes
import os

from .errors import STATUS, NativeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libboxscreen_b200.so")

BX_F64, BX_F32 = 0, 1
BX_PG, BX_CD, BX_APG, BX_ACTIVE_SET = 0, 1, 2, 3
KINDS = {"pg": BX_PG, "cd": BX_CD, "apg": BX_APG, "active-set": BX_ACTIVE_SET}
RESTARTS = {"adaptive": 0, "function": 1}


class SolveCfg(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("inner_passes", ctypes.c_int32),
                ("max_rounds", ctypes.c_int64), ("gap_tol", ctypes.c_double),
                ("step_size", ctypes.c_double), ("power_iters", ctypes.c_int32),
                ("screening", ctypes.c_int32), ("alpha", ctypes.c_double),
                ("slack_scale", ctypes.c_double), ("relative_gap", ctypes.c_int32),
                ("restart", ctypes.c_int32)]


class TraceRec(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int64), ("elapsed", ctypes.c_double),
                ("primal", ctypes.c_double), ("dual", ctypes.c_double), ("gap", ctypes.c_double),
                ("preserved_count", ctypes.c_int64), ("newly_screened_lower", ctypes.c_int64),
                ("newly_screened_upper", ctypes.c_int64), ("eps", ctypes.c_double),
                ("radius", ctypes.c_double), ("step", ctypes.c_double),
                ("certified_gap", ctypes.c_double), ("restarts", ctypes.c_int64), ("momentum", ctypes.c_double)]


class SolveOut(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("converged", ctypes.c_int32), ("gap", ctypes.c_double),
                ("n_sat_lower", ctypes.c_int64), ("n_sat_upper", ctypes.c_int64),
                ("iterations", ctypes.c_int64), ("step", ctypes.c_double), ("sigma", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64), ("restarts", ctypes.c_int64),
                ("spec_kept", ctypes.c_int64), ("spec_undone", ctypes.c_int64)]


class ProfEntry(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("ms", ctypes.c_double), ("bytes", ctypes.c_double)]


PROF_SLOTS = 13
PROF_NAMES = ["pass_dot", "pass_pg_g", "pass_pg", "pass_apg", "pass_power", "pass_ax", "reduce", "dual",
              "sphere", "gather", "cd", "active", "small_round"]

class BatchedOut(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("converged", ctypes.c_int64), ("iterations", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("max_gap", ctypes.c_double),
                ("sphere_sweeps", ctypes.c_int64), ("tiles", ctypes.c_int64), ("round_kernel_ms", ctypes.c_double)]


START_FN = ctypes.CFUNCTYPE(None, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                            ctypes.c_void_p)

# every symbol include/boxscreen_b200.h declares, with (restype, argtypes)
_vp, _i32, _i64, _d, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
_dp = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "bx_workspace_bytes": (_sz, [_i64, _i64, _i32]),
    "bx_ctx_create": (ctypes.c_int, [ctypes.POINTER(_vp), _i64, _i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp,
                                     _vp, _sz, _vp]),
    "bx_ctx_destroy": (ctypes.c_int, [_vp]),
    "bx_last_error": (ctypes.c_char_p, [_vp]),
    "bx_col_norms": (ctypes.c_int, [_vp, _vp]),
    "bx_att": (ctypes.c_int, [_vp, _vp]),
    "bx_power_iter": (ctypes.c_int, [_vp, _i32, _dp, _dp]),
    "bx_reset": (ctypes.c_int, [_vp]),
    "bx_primal_passes": (ctypes.c_int, [_vp, _i32, _d, _i32]),
    "bx_dual_screen": (ctypes.c_int, [_vp, _i32, _d, _d, _dp]),
    "bx_compact": (ctypes.c_int, [_vp]),
    "bx_certified_gap": (ctypes.c_int, [_vp, _d, _dp]),
    "bx_set_state": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64), _i64, _vp, _vp]),
    "bx_gradient": (ctypes.c_int, [_vp, _vp, _vp]),
    "bx_active_set_step": (ctypes.c_int, [_vp, _vp, _vp, ctypes.POINTER(ctypes.c_int32)]),
    "bx_apply_a": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "bx_apply_at": (ctypes.c_int, [_vp, _vp, _vp]),
    "bx_dual_point": (ctypes.c_int, [_vp, _vp, _d, _vp, _vp, _dp]),
    "bx_eval_dual": (ctypes.c_int, [_vp, _vp, _vp, _dp]),
    "bx_sphere_test": (ctypes.c_int, [_vp, _vp, _vp, _i64, _d, _d, _vp]),
    "bx_preserved_count": (_i64, [_vp]),
    "bx_solve": (ctypes.c_int, [_vp, ctypes.POINTER(SolveCfg), START_FN, _vp, ctypes.POINTER(TraceRec), _i64,
                                ctypes.POINTER(SolveOut)]),
    "bx_get_state": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "bx_get_prev_iterate": (ctypes.c_int, [_vp, _vp]),
    "bx_active_set_workspace_bytes": (_sz, [_i64, _i64]),
    "bx_ctx_set_active_set_workspace": (ctypes.c_int, [_vp, _vp, _sz]),
    "bx_peer_alloc": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "bx_peer_open": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "bx_peer_disable": (ctypes.c_int, [_vp]),
    "bx_comm_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_char_p, _i32, _i32]),
    "bx_comm_destroy": (ctypes.c_int, [_vp]),
    "bx_comm_peer_alloc": (ctypes.c_int, [_vp, _i64, ctypes.c_char_p]),
    "bx_comm_peer_open": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "bx_comm_peer_disable": (ctypes.c_int, [_vp]),
    "bx_ctx_use_comm": (ctypes.c_int, [_vp, _vp, _i64, _i64]),
    "bx_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "bx_ctx_set_comm": (ctypes.c_int, [_vp, ctypes.c_char_p, _i32, _i32, _i64, _i64]),
    "bx_group_create": (ctypes.c_int, [ctypes.POINTER(_vp), _i32]),
    "bx_group_destroy": (ctypes.c_int, [_vp]),
    "bx_ctx_set_group": (ctypes.c_int, [_vp, _vp, _i32, _i64, _i64]),
    "bx_set_profiling": (ctypes.c_int, [_vp, _i32]),
    "bx_get_profile": (ctypes.c_int, [_vp, ctypes.POINTER(ProfEntry), _i32]),
    "bx_batched_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "bx_batched_create": (ctypes.c_int, [ctypes.POINTER(_vp), _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _sz,
                                         _vp]),
    "bx_batched_run": (ctypes.c_int, [_vp, _d, _i32, _i32, _i32, _d, _dp, _i64, ctypes.POINTER(BatchedOut)]),
    "bx_batched_set_check_every": (ctypes.c_int, [_vp, _i32]),
    "bx_batched_run_to_host": (ctypes.c_int, [_vp, _d, _i32, _i32, _i32, _d, _dp, _i64, ctypes.POINTER(BatchedOut),
                                              _vp, _i64]),
    "bx_batched_get": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "bx_batched_last_error": (ctypes.c_char_p, [_vp]),
    "bx_batched_destroy": (ctypes.c_int, [_vp]),
}

_lib = None


def lib():
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library {LIB_PATH} not built; run `python -m paper_2202_07258_b200.build` "
                "(there is no CPU fallback)")
        h = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status, ctx=None, what=""):
    if status == 0:
        return
    msg = ""
    if ctx is not None:
        raw = lib().bx_last_error(ctx)
        msg = raw.decode() if raw else ""
    exc = STATUS.get(status, NativeError)
    raise exc(f"{what}: {msg}" if what else msg)

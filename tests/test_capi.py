"""The C-ABI library loads and exports every symbol include/boxscreen_b200.h
declares (CPU only: no compute calls), and the host-side logic that needs no
GPU behaves like the reference."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "boxscreen_b200.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:int|size_t|int64_t|const char\s*\*)\s+(bx_\w+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("bx_ctx_create", "bx_ctx_destroy", "bx_solve", "bx_get_state", "bx_certified_gap",
                 "bx_power_iter", "bx_compact", "bx_dual_screen", "bx_primal_passes", "bx_ctx_set_comm"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2202_07258_b200 import _native as nat
    lib = nat.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in nat.SIGNATURES, f"{name} has no ctypes signature"


def test_workspace_sizing_is_host_only():
    from paper_2202_07258_b200 import _native as nat
    b64 = nat.lib().bx_workspace_bytes(10000, 50000, nat.BX_F64)
    b32 = nat.lib().bx_workspace_bytes(10000, 50000, nat.BX_F32)
    # A_act copy dominates: m_pad * n * elem
    assert 4.0e9 <= b64 <= 4.3e9
    assert 2.0e9 <= b32 <= 2.2e9


def test_problem_validation_matches_reference():
    from paper_2202_07258_b200 import Problem
    from paper_2202_07258_b200.errors import DimensionMismatch
    with pytest.raises(DimensionMismatch):
        Problem(np.ones((3, 2)), np.ones(2), 0.0, 1.0)
    with pytest.raises(ValueError):
        Problem(np.ones((2, 2)), np.ones(2), 1.0, 1.0)
    with pytest.raises(ValueError):
        Problem(np.ones((2, 2)), np.ones(2), -np.inf, 1.0)
    with pytest.raises(ValueError):
        Problem(np.array([[np.nan, 1.0], [1.0, 1.0]]), np.ones(2), 0.0, 1.0)
    p = Problem(np.ones((2, 3)), np.ones(2), 0.0, [1.0, np.inf, 2.0])
    assert list(p.j_inf) == [1]
    assert not p.a_matrix.flags.writeable


def test_solver_config_validation():
    from paper_2202_07258_b200 import SolverConfig
    with pytest.raises(ValueError):
        SolverConfig(kind="newton")
    with pytest.raises(ValueError):
        SolverConfig(gap_tol=0.0)
    with pytest.raises(ValueError):
        SolverConfig(inner_passes=0)
    assert SolverConfig(kind="apg").kind == "apg"


def test_radius_and_clamp():
    from paper_2202_07258_b200 import clamp_gap, gap_safe_radius
    from paper_2202_07258_b200.errors import InternalConsistency, NegativeGap
    assert gap_safe_radius(0.0, 1.0) == 0.0
    assert gap_safe_radius(2.0, 1.0) == 2.0
    assert gap_safe_radius(1.0, 2.0) == 1.0
    with pytest.raises(NegativeGap):
        gap_safe_radius(-1e-12, 1.0)
    assert clamp_gap(-1e-10) == 0.0
    with pytest.raises(InternalConsistency):
        clamp_gap(-1e-8)


def test_trace_csv_format(tmp_path):
    from paper_2202_07258_b200 import TraceRecord, trace_to_csv
    tr = [TraceRecord(1, 0.5, 1.0, 0.5, 0.5, 3, 0.25, 1, 0)]
    path = tmp_path / "t.csv"
    trace_to_csv(tr, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "round,elapsed_s,primal,dual,gap,preserved,ratio"
    assert lines[1] == "1,0.500000000,1,0.5,0.5,3,0.25"


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    with pytest.raises(RuntimeError):
        solve(Problem(np.eye(2), np.ones(2), 0.0, 1.0), SolverConfig(kind="pg"))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2202_07258_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from\s+oracle|import\s+oracle)|__import__\(.oracle|#include.*oracle",
                                     src, flags=re.M), f

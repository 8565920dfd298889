"""The C-ABI library loads and exports every symbol include/fcgno.h declares; host-only
queries and argument validation behave as documented (no GPU needed, no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcgno.h")


@pytest.fixture(scope="module")
def built():
    from paper_2402_05598_b200 import build
    return build.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fcgno_[a-zA-Z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("fcgno_assemble", "fcgno_apply_A", "fcgno_apply_NO", "fcgno_fcg_solve"):
        assert required in names


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(built)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol(built):
    from paper_2402_05598_b200 import fcgno
    assert set(declared_functions()) <= set(fcgno.EXPORTS)
    assert fcgno.abi_version() == 9


def test_sizes_and_validation(built):
    from paper_2402_05598_b200 import fcgno as F
    import synthetic as sy
    g = F.Grid(64, 4)
    assert F._lib.fcgno_problem_workspace_bytes(g) > 0
    assert F._lib.fcgno_problem_workspace_bytes(F.Grid(1, 4)) == 0
    for w in (32, 48, 85):
        d32 = F.NoDesc(w, F.FP32, 1)
        d64 = F.NoDesc(w, F.FP64, 1)
        b32 = F._lib.fcgno_no_packed_bytes(d32)
        assert F._lib.fcgno_no_packed_bytes(d64) == 2 * b32
        # folded layout is smaller than the canonical blob (layer 4 + lift folded)
        assert b32 // 4 < sy.no_blob_size(w)
    assert F._lib.fcgno_no_packed_bytes(F.NoDesc(0, F.FP32, 1)) == 0
    ok = F.SolveOpts(5, 100, 1e-6, F.SCHEDULE_PAPER, 16, 0)
    assert F._lib.fcgno_solve_workspace_bytes(g, None, ok) > 0
    for bad in (F.SolveOpts(0, 100, 1e-6, 0, 16, 0), F.SolveOpts(65, 100, 1e-6, 0, 16, 0),
                F.SolveOpts(5, -1, 1e-6, 0, 16, 0), F.SolveOpts(5, 10, 1e-6, 7, 16, 0)):
        assert F._lib.fcgno_solve_workspace_bytes(g, None, bad) == 0
    # solve workspace grows with m (ring of m+1 (p, s) pairs)
    v32 = F._lib.fcgno_solve_workspace_bytes(g, None, F.SolveOpts(5, 10, 1e-6, 0, 16, 0, 1))
    v64 = F._lib.fcgno_solve_workspace_bytes(g, None, F.SolveOpts(5, 10, 1e-6, 0, 16, 0, 0))
    assert 0 < v32 < v64                                  # fp32 vectors and ring (R21)
    assert F._lib.fcgno_solve_workspace_bytes(g, None, F.SolveOpts(5, 10, 1e-6, 0, 16, 0, 2)) == 0
    a = F._lib.fcgno_solve_workspace_bytes(g, None, F.SolveOpts(5, 10, 1e-6, 0, 16, 0))
    b = F._lib.fcgno_solve_workspace_bytes(g, None, F.SolveOpts(10, 10, 1e-6, 0, 16, 0))
    assert b - a >= 2 * 5 * 4 * 64 * 64 * 8
    # NULL arguments are rejected before any CUDA call
    assert F._lib.fcgno_assemble(g, None, None, 0, None, None) == 1
    assert b"NULL" in F._lib.fcgno_last_error()
    assert F._lib.fcgno_apply_A(None, None, None, None) == 1


def test_profile_api(built):
    from paper_2402_05598_b200 import fcgno as F
    F.profile_reset()
    prof = F.profile_read()
    assert len(prof) == F.PROF_NCLASS and prof["k_no_layer"] == (0.0, 0)

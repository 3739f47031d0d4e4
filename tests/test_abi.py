"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol that
include/mstrsm.h declares, and rejects invalid arguments (LAPACK INFO style, -i) or returns 0 for
empty problems before touching CUDA."""
import ctypes
import os
import re

import pytest

import paper_1607_01477_b200 as ms

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mstrsm.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while")))


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for required in ["mstrsm_d", "mstrsm_z", "mstrsm_d_safe", "mstrsm_z_safe", "mstrsm_d_ex", "mstrsm_z_ex",
                     "trevc_d", "trevc_z", "trevc_d_cols", "trevc_z_cols", "trevc_z_host", "pseudospectra_z",
                     "mstrsm_set_stream", "mstrsm_get_stream", "mstrsm_error_string", "mstrsm_status",
                     "mstrsm_launch_count", "mstrsm_fp64_peak", "mstrsm_d_gen", "mstrsm_z_gen", "tgevc_d",
                     "tgevc_z", "eig_backtransform_d", "eig_backtransform_z", "trevc_qz_d", "trevc_qz_z",
                     "mstrsm_comm_init", "mstrsm_comm_destroy", "trevc_z_dist", "mstrsm_workspace_size"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(ms.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    """The shipped cubin targets sm_100a (cuobjdump lists the ELF arch)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", ms.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _lib():
    return ms.load()


def test_invalid_arguments_are_rejected_without_cuda():
    lib = _lib()
    P = None
    # mstrsm_d(U, ldu, m, shifts, B, ldb, n, scales, nb)
    assert lib.mstrsm_d(P, 1, -1, P, P, 1, 1, P, 32) == -3      # m < 0
    assert lib.mstrsm_d(P, 3, 4, P, P, 4, 1, P, 32) == -2       # ldu < m
    assert lib.mstrsm_d(P, 4, 4, P, P, 3, 1, P, 32) == -6       # ldb < m
    assert lib.mstrsm_d(P, 4, 4, P, P, 4, -2, P, 32) == -7      # n < 0
    assert lib.mstrsm_d(P, 4, 4, P, P, 4, 1, P, 129) == -9      # nb > 128
    assert lib.mstrsm_d(P, 4, 4, P, P, 4, 1, P, -1) == -9       # nb < 0
    assert lib.mstrsm_d(P, 4, 4, P, P, 4, 1, P, 0) == -1        # U NULL
    assert lib.mstrsm_d_safe(ctypes.c_void_p(8), 4, 4, ctypes.c_void_p(8), ctypes.c_void_p(8), 4, 1, P, 32) == -8
    # mstrsm_z_ex(safe, op, U, ldu, m, shifts, stride, B, ldb, n, row_end, scales, exp, nb)
    assert lib.mstrsm_z_ex(2, 0, P, 4, 4, P, 1, P, 4, 1, P, P, P, 0) == -1
    assert lib.mstrsm_z_ex(0, 5, P, 4, 4, P, 1, P, 4, 1, P, P, P, 0) == -2
    re_ = (ctypes.c_int64 * 1)(3)
    assert lib.mstrsm_z_ex(0, 1, P, 4, 4, P, 1, P, 4, 1, re_, P, P, 0) == -11   # row_end with op C
    # trevc_z(T, ldt, m, Z, ldz, scales, exp, nb)
    assert lib.trevc_z(P, 2, 3, P, 3, P, P, 0) == -2
    assert lib.trevc_z(P, 3, 3, P, 2, P, P, 0) == -5
    assert lib.trevc_z(P, 3, 3, P, 3, P, P, 200) == -8
    # pseudospectra_z(U, ldu, m, z, npts, iters, v0, sigma, flags, nb)
    assert lib.pseudospectra_z(P, 4, 4, P, 1, 0, P, P, P, 0) == -6
    # mstrsm_z_side(safe, side, uplo, A, lda, m, shifts, stride, B, ldb, n, scales, exp, nb)  (§8f f4)
    assert lib.mstrsm_z_side(0, 2, 0, P, 4, 4, P, 1, P, 4, 1, P, P, 0) == -2
    assert lib.mstrsm_z_side(0, 1, 0, P, 4, 4, P, 1, P, 1, 3, P, P, 0) == -10     # right: ldb >= n
    assert lib.mstrsm_d_side(0, 0, 1, P, 3, 4, P, 1, P, 4, 1, P, P, 0) == -5
    assert lib.mstrsm_d_side(1, 0, 1, ctypes.c_void_p(8), 4, 4, ctypes.c_void_p(8), 1, ctypes.c_void_p(8), 4, 1,
                             P, P, 0) == -12                                      # safe needs scales
    # spectral_cloud_z(U, ldu, m, z, npts, maxit, tol, v0, sigma, flags, its, nb)
    assert lib.spectral_cloud_z(P, 4, 4, P, 1, 15, ctypes.c_double(-1.0), P, P, P, P, 0) == -7
    assert lib.spectral_cloud_z(P, 4, 4, P, 1, 0, ctypes.c_double(0.0), P, P, P, P, 0) == -6
    assert lib.spectral_window_z(P, 4, 4, ctypes.c_double(0), ctypes.c_double(1), -1, ctypes.c_double(0),
                                 ctypes.c_double(1), 2, 15, ctypes.c_double(0), P, P, P, P, 0) == -6
    assert lib.spectral_portrait_z(P, 3, 4, 2, 2, 15, ctypes.c_double(0), P, P, P, P, P, 0) == -2
    # eig_backtransform_z(Q, ldq, m, Z, ldz, n, cols, X, ldx)
    assert lib.eig_backtransform_z(P, 3, 4, P, 4, 4, P, P, 4) == -2
    assert lib.eig_backtransform_z(P, 4, 4, P, 4, 5, P, P, 4) == -6      # n > m without row bounds
    assert lib.eig_backtransform_d(P, 4, 4, P, 4, 4, P, P, 3) == -9
    bad = (ctypes.c_int64 * 2)(2, 2)
    assert lib.eig_backtransform_d(ctypes.c_void_p(8), 4, 4, ctypes.c_void_p(8), 4, 2, bad, ctypes.c_void_p(8), 4) == -7
    # trevc_qz_z(T, ldt, m, Q, ldq, X, ldx, scales, exp, nb)
    assert lib.trevc_qz_z(P, 4, 4, P, 3, P, 4, P, P, 0) == -5
    assert lib.trevc_qz_d(P, 4, 4, P, 4, P, 4, P, P, 129) == -10


def test_empty_problems_return_zero_without_cuda():
    lib = _lib()
    P = None
    assert lib.mstrsm_z(P, 1, 0, P, P, 1, 5, P, 0) == 0
    assert lib.mstrsm_d_safe(P, 4, 4, P, P, 4, 0, P, 0) == 0
    assert lib.trevc_d(P, 1, 0, P, 1, P, P, 0) == 0
    assert lib.pseudospectra_z(P, 1, 0, P, 0, 15, P, P, P, 0) == 0
    assert lib.eig_backtransform_z(P, 1, 0, P, 1, 0, P, P, 1) == 0
    assert lib.trevc_qz_d(P, 1, 0, P, 1, P, 1, P, P, 0) == 0


def test_workspace_size_without_cuda():
    lib = _lib()
    small = lib.mstrsm_workspace_size(100, 10, 32, 0, 1)
    big = lib.mstrsm_workspace_size(1000, 100, 32, 1, 1)
    assert 0 < small < big
    assert lib.mstrsm_workspace_size(100, 10, 200, 0, 1) == 0          # invalid nb
    assert lib.mstrsm_workspace_size(0, 10, 32, 0, 1) == 0             # empty problem
    assert lib.mstrsm_z_ex_ws(0, 0, None, 4, 4, None, 1, None, 4, 1, None, None, None, 0,
                              ctypes.c_void_p(256), 1) == -3               # U NULL, checked before CUDA


def test_error_strings():
    lib = _lib()
    assert lib.mstrsm_error_string(0) == b"success"
    assert b"non-finite" in lib.mstrsm_error_string(2)
    assert b"invalid" in lib.mstrsm_error_string(-3)


def test_no_cpu_fallback_without_cuda():
    """Calling the product path without a GPU raises; it never computes on the CPU."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    U = torch.from_numpy(np.eye(4))
    with pytest.raises(ms.MstrsmError):
        ms.solve(U, torch.zeros(1, dtype=torch.float64), torch.ones(4, 1, dtype=torch.float64))


def test_sync_status_switch_needs_no_gpu():
    lib = ctypes.CDLL(ms.LIB_PATH)
    assert lib.mstrsm_set_sync_status(1) == 0
    assert lib.mstrsm_set_sync_status(0) == 0

"""ctypes binding for libmstrsm.so (C ABI in include/mstrsm.h).

Argument marshalling only: every step of the solve runs in the library's sm_100a kernels.
Functions carry the C names (``mstrsm_d``, ``mstrsm_z_safe``, ``trevc_z``, ``pseudospectra_z``,
...) and take torch CUDA tensors; a few convenience wrappers (``solve``, ``trevc``,
``pseudospectra``) allocate outputs.  The library runs on torch's current CUDA stream.

There is no CPU fallback: if the library is missing or CUDA is unavailable, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSTRSM_LIB", os.path.join(_HERE, "libmstrsm.so"))   # override: experiments only
_lib = None

c_i64, c_int, c_dbl, c_vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p

__all__ = [
    "load", "LIB_PATH", "MstrsmError",
    "mstrsm_d", "mstrsm_z", "mstrsm_d_safe", "mstrsm_z_safe", "mstrsm_d_ex", "mstrsm_z_ex",
    "trevc_d", "trevc_z", "trevc_d_cols", "trevc_z_cols", "trevc_z_host", "trevc_z_host_batch", "pseudospectra_z",
    "mstrsm_d_gen", "mstrsm_z_gen", "tgevc_d", "tgevc_z", "solve_gen", "tgevc",
    "spectral_cloud_z", "spectral_window_z", "spectral_portrait_z", "spectral_cloud", "spectral_window",
    "spectral_portrait", "comm_init", "comm_destroy", "dist_shard", "trevc_dist", "solve_dist", "pack_cols", "unpack_cols", "mstrsm_workspace_size", "mstrsm_d_ex_ws", "mstrsm_z_ex_ws", "mstrsm_d_side", "mstrsm_z_side", "solve_side",
    "eig_backtransform_d", "eig_backtransform_z", "trevc_qz_d", "trevc_qz_z", "eig_backtransform", "trevc_qz",
    "mstrsm_status", "mstrsm_set_sync_status", "mstrsm_launch_count", "mstrsm_fp64_peak", "mstrsm_error_string",
    "mstrsm_profile", "mstrsm_profile_read", "mstrsm_gemm_real_products",
    "solve", "trevc", "pseudospectra", "fp64_peak", "status", "launch_count", "gemm_real_products",
]


class MstrsmError(RuntimeError):
    pass


def load():
    """Load libmstrsm.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MstrsmError(f"{LIB_PATH} not built; run `make` or __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    P = c_vp
    sig = {
        "mstrsm_d": [P, c_i64, c_i64, P, P, c_i64, c_i64, P, c_int],
        "mstrsm_z": [P, c_i64, c_i64, P, P, c_i64, c_i64, P, c_int],
        "mstrsm_d_safe": [P, c_i64, c_i64, P, P, c_i64, c_i64, P, c_int],
        "mstrsm_z_safe": [P, c_i64, c_i64, P, P, c_i64, c_i64, P, c_int],
        "mstrsm_d_ex": [c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, P, c_int],
        "mstrsm_z_ex": [c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, P, c_int],
        "trevc_d": [P, c_i64, c_i64, P, c_i64, P, P, c_int],
        "trevc_z": [P, c_i64, c_i64, P, c_i64, P, P, c_int],
        "trevc_d_cols": [P, c_i64, c_i64, P, c_i64, P, c_i64, P, P, c_int],
        "trevc_z_cols": [P, c_i64, c_i64, P, c_i64, P, c_i64, P, P, c_int],
        "trevc_z_host": [P, c_i64, c_i64, P, c_i64, P, P, c_int],
        "trevc_z_host_batch": [P, c_i64, c_i64, P, c_i64, P, P, c_i64, c_int],
        "pseudospectra_z": [P, c_i64, c_i64, P, c_i64, c_int, P, P, P, c_int],
        "mstrsm_comm_unique_id": [P],
        "mstrsm_d_pack_cols": [P, c_i64, c_i64, P, P, P, P],
        "mstrsm_z_pack_cols": [P, c_i64, c_i64, P, P, P, P],
        "mstrsm_d_unpack_cols": [P, c_i64, P, P, P, c_i64, P, c_i64],
        "mstrsm_z_unpack_cols": [P, c_i64, P, P, P, c_i64, P, c_i64],
        "mstrsm_comm_init": [c_int, c_int, P],
        "mstrsm_comm_destroy": [],
        "trevc_d_dist": [P, c_i64, c_i64, P, c_i64, P, P, c_int, c_int],
        "mstrsm_d_dist": [c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, c_int, c_int],
        "mstrsm_z_dist": [c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, c_int, c_int],
        "trevc_z_dist": [P, c_i64, c_i64, P, c_i64, P, P, c_int, c_int],
        "mstrsm_d_ex_ws": [c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, P, c_int, P,
                           ctypes.c_size_t],
        "mstrsm_z_ex_ws": [c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, P, c_int, P,
                           ctypes.c_size_t],
        "mstrsm_d_side": [c_int, c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, c_int],
        "mstrsm_z_side": [c_int, c_int, c_int, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, c_int],
        "spectral_cloud_z": [P, c_i64, c_i64, P, c_i64, c_int, c_dbl, P, P, P, P, c_int],
        "spectral_window_z": [P, c_i64, c_i64, c_dbl, c_dbl, c_i64, c_dbl, c_dbl, c_i64, c_int, c_dbl, P, P, P, P,
                              c_int],
        "spectral_portrait_z": [P, c_i64, c_i64, c_i64, c_i64, c_int, c_dbl, P, P, P, P, P, c_int],
        "mstrsm_d_gen": [c_int, P, c_i64, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, P, c_int],
        "mstrsm_z_gen": [c_int, P, c_i64, P, c_i64, c_i64, P, c_i64, P, c_i64, c_i64, P, P, P, c_int],
        "tgevc_d": [P, c_i64, P, c_i64, c_i64, P, c_i64, P, P, P, c_int],
        "tgevc_z": [P, c_i64, P, c_i64, c_i64, P, c_i64, P, P, P, c_int],
        "eig_backtransform_d": [P, c_i64, c_i64, P, c_i64, c_i64, P, P, c_i64],
        "eig_backtransform_z": [P, c_i64, c_i64, P, c_i64, c_i64, P, P, c_i64],
        "trevc_qz_d": [P, c_i64, c_i64, P, c_i64, P, c_i64, P, P, c_int],
        "trevc_qz_z": [P, c_i64, c_i64, P, c_i64, P, c_i64, P, P, c_int],
        "mstrsm_set_stream": [P],
        "mstrsm_status": [],
        "mstrsm_set_sync_status": [c_int],
        "mstrsm_launch_count": [c_int],
        "mstrsm_fp64_peak": [c_dbl, P, P],
        "mstrsm_error_string": [c_int],
        "mstrsm_profile": [c_int],
        "mstrsm_profile_read": [c_int, P, P, P],
        "mstrsm_gemm_real_products": [],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = c_int
    lib.mstrsm_launch_count.restype = c_i64
    lib.mstrsm_dist_shard.restype = c_i64
    lib.mstrsm_dist_shard.argtypes = [c_i64, c_int, c_int, P]
    lib.mstrsm_workspace_size.restype = ctypes.c_size_t
    lib.mstrsm_workspace_size.argtypes = [c_i64, c_i64, c_int, c_int, c_int]
    lib.mstrsm_error_string.restype = ctypes.c_char_p
    lib.mstrsm_get_stream.restype = c_vp
    _lib = lib
    return lib


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise MstrsmError("CUDA is not available: libmstrsm has no CPU path")
    return torch


def _bind_stream(lib):
    torch = _torch()
    lib.mstrsm_set_stream(c_vp(torch.cuda.current_stream().cuda_stream))


def _check(rc: int, name: str):
    if rc != 0:
        msg = _lib.mstrsm_error_string(rc).decode()
        raise MstrsmError(f"{name} returned {rc}: {msg}")


def _ptr(t):
    if t is None:
        return None
    return c_vp(t.data_ptr())


def _ld(t) -> int:
    """Leading dimension of a column-major (Fortran-strided) 2-D tensor."""
    if t.dim() == 1:
        return max(1, t.shape[0])
    if t.stride(0) != 1:
        raise ValueError("matrices must be column-major: use tensor.t().contiguous().t() "
                         "or allocate with torch.empty(n, m).t()")
    return max(1, t.stride(1), t.shape[0])


def _host_i64(a):
    if a is None:
        return None, None
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    return arr, arr.ctypes.data_as(c_vp)


def _row_end(a, n):
    """row_end for the C call: a CUDA int64 tensor is passed as a device pointer (the ABI's form,
    include/mstrsm.h), anything else is converted to a host int64 array."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor) and a.is_cuda:
            if a.dtype != torch.int64 or not a.is_contiguous() or a.numel() < n:
                raise ValueError("row_end: a contiguous int64 CUDA tensor with at least n entries")
            return a, c_vp(a.data_ptr())
    except ImportError:
        pass
    arr, p = _host_i64(a)
    if arr.size < n:
        raise ValueError("row_end: at least n entries")
    return arr, p


# ------------------------------------------------------------------ C-named entry points
def _call(name, *args):
    lib = load()
    _bind_stream(lib)
    _check(getattr(lib, name)(*args), name)


def mstrsm_d(U, ldu, m, shifts, B, ldb, n, scales, nb):
    _call("mstrsm_d", _ptr(U), ldu, m, _ptr(shifts), _ptr(B), ldb, n, _ptr(scales), nb)


def mstrsm_z(U, ldu, m, shifts, B, ldb, n, scales, nb):
    _call("mstrsm_z", _ptr(U), ldu, m, _ptr(shifts), _ptr(B), ldb, n, _ptr(scales), nb)


def mstrsm_d_safe(U, ldu, m, shifts, B, ldb, n, scales, nb):
    _call("mstrsm_d_safe", _ptr(U), ldu, m, _ptr(shifts), _ptr(B), ldb, n, _ptr(scales), nb)


def mstrsm_z_safe(U, ldu, m, shifts, B, ldb, n, scales, nb):
    _call("mstrsm_z_safe", _ptr(U), ldu, m, _ptr(shifts), _ptr(B), ldb, n, _ptr(scales), nb)


def mstrsm_d_ex(safe, op, U, ldu, m, shifts, shift_stride, B, ldb, n, row_end, scales, scale_exp, nb):
    arr, p = _row_end(row_end, n)
    _call("mstrsm_d_ex", safe, op, _ptr(U), ldu, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n, p,
          _ptr(scales), _ptr(scale_exp), nb)


def mstrsm_z_ex(safe, op, U, ldu, m, shifts, shift_stride, B, ldb, n, row_end, scales, scale_exp, nb):
    arr, p = _row_end(row_end, n)
    _call("mstrsm_z_ex", safe, op, _ptr(U), ldu, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n, p,
          _ptr(scales), _ptr(scale_exp), nb)


def trevc_d(T, ldt, m, Z, ldz, scales, scale_exp, nb):
    _call("trevc_d", _ptr(T), ldt, m, _ptr(Z), ldz, _ptr(scales), _ptr(scale_exp), nb)


def trevc_z(T, ldt, m, Z, ldz, scales, scale_exp, nb):
    _call("trevc_z", _ptr(T), ldt, m, _ptr(Z), ldz, _ptr(scales), _ptr(scale_exp), nb)


def trevc_d_cols(T, ldt, m, cols_host, ncols, Z, ldz, scales, scale_exp, nb):
    arr, p = _host_i64(cols_host)
    _call("trevc_d_cols", _ptr(T), ldt, m, p, ncols, _ptr(Z), ldz, _ptr(scales), _ptr(scale_exp), nb)


def trevc_z_cols(T, ldt, m, cols_host, ncols, Z, ldz, scales, scale_exp, nb):
    arr, p = _host_i64(cols_host)
    _call("trevc_z_cols", _ptr(T), ldt, m, p, ncols, _ptr(Z), ldz, _ptr(scales), _ptr(scale_exp), nb)


def _check_host_square(A, m: int, name: str) -> int:
    """A host matrix the C ABI reads as column-major complex128 with leading dimension
    A.shape[0] >= m and at least m columns; returns that leading dimension."""
    if not isinstance(A, np.ndarray):
        raise TypeError(f"{name} must be a numpy array")
    if A.dtype != np.complex128:
        raise TypeError(f"{name} must be complex128 (got {A.dtype})")
    if A.ndim != 2 or not A.flags.f_contiguous:
        raise ValueError(f"{name} must be a 2-D Fortran-ordered (column-major) array")
    if A.shape[0] < max(1, m) or A.shape[1] < m:
        raise ValueError(f"{name} has shape {A.shape}; need at least ({m}, {m})")
    return int(A.shape[0])


def _check_host_vec(v, m: int, dtype, name: str):
    if v is None:
        return
    if not isinstance(v, np.ndarray) or v.dtype != dtype or v.ndim != 1 or not v.flags.c_contiguous:
        raise TypeError(f"{name} must be a contiguous 1-D numpy {np.dtype(dtype).name} array")
    if v.shape[0] < m:
        raise ValueError(f"{name} has length {v.shape[0]}; need at least {m}")


def trevc_z_host(T_host: np.ndarray, m: int, Z_host: np.ndarray, scales_host=None, exp_host=None, nb=0):
    """Host-buffer end-to-end entry (numpy complex128 Fortran arrays, blocking).  The arrays are
    checked here (dtype, column-major order, shape, lengths) because the C ABI reads and writes
    them through raw pointers."""
    ldt = _check_host_square(T_host, m, "T_host")
    ldz = _check_host_square(Z_host, m, "Z_host")
    if not Z_host.flags.writeable:
        raise ValueError("Z_host must be writeable")
    _check_host_vec(scales_host, m, np.float64, "scales_host")
    _check_host_vec(exp_host, m, np.int32, "exp_host")
    lib = load()
    _bind_stream(lib)
    ptr = lambda a: a.ctypes.data_as(c_vp) if a is not None else None
    _check(lib.trevc_z_host(ptr(T_host), ldt, m, ptr(Z_host), ldz, ptr(scales_host), ptr(exp_host), nb),
           "trevc_z_host")


def trevc_z_host_batch(T_hosts, m: int, Z_hosts, scales_hosts=None, exp_hosts=None, nb=0):
    """Batched host-buffer entry (lists of numpy complex128 Fortran arrays, blocking): problem
    k's solve overlaps k+1's upload and k-1's download.  Every problem must share one leading
    dimension for T and one for Z (the C ABI takes one ldt and one ldz)."""
    n = len(T_hosts)
    if len(Z_hosts) != n:
        raise ValueError("T_hosts and Z_hosts must have the same length")
    for lst, nm in ((scales_hosts, "scales_hosts"), (exp_hosts, "exp_hosts")):
        if lst is not None and len(lst) != n:
            raise ValueError(f"{nm} must have one entry per problem")
    ldt = ldz = 1
    for k in range(n):
        lt = _check_host_square(T_hosts[k], m, f"T_hosts[{k}]")
        lz = _check_host_square(Z_hosts[k], m, f"Z_hosts[{k}]")
        if not Z_hosts[k].flags.writeable:
            raise ValueError(f"Z_hosts[{k}] must be writeable")
        if k == 0:
            ldt, ldz = lt, lz
        elif lt != ldt or lz != ldz:
            raise ValueError("every problem of a batch must have the same leading dimensions")
        _check_host_vec(scales_hosts[k] if scales_hosts is not None else None, m, np.float64, f"scales_hosts[{k}]")
        _check_host_vec(exp_hosts[k] if exp_hosts is not None else None, m, np.int32, f"exp_hosts[{k}]")
    lib = load()
    _bind_stream(lib)
    arr = lambda lst: (c_vp * n)(*[a.ctypes.data if a is not None else None for a in lst]) if lst is not None else None
    _check(lib.trevc_z_host_batch(arr(T_hosts), ldt, m, arr(Z_hosts), ldz, arr(scales_hosts), arr(exp_hosts), n, nb),
           "trevc_z_host_batch")


def mstrsm_d_gen(safe, U, ldu, V, ldv, m, shifts, shift_stride, B, ldb, n, row_end, scales, scale_exp, nb):
    arr, p = _row_end(row_end, n)
    _call("mstrsm_d_gen", safe, _ptr(U), ldu, _ptr(V), ldv, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n, p,
          _ptr(scales), _ptr(scale_exp), nb)


def mstrsm_z_gen(safe, U, ldu, V, ldv, m, shifts, shift_stride, B, ldb, n, row_end, scales, scale_exp, nb):
    arr, p = _row_end(row_end, n)
    _call("mstrsm_z_gen", safe, _ptr(U), ldu, _ptr(V), ldv, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n, p,
          _ptr(scales), _ptr(scale_exp), nb)


def tgevc_d(T, ldt, S, lds, m, Z, ldz, lam, scales, scale_exp, nb):
    _call("tgevc_d", _ptr(T), ldt, _ptr(S), lds, m, _ptr(Z), ldz, _ptr(lam), _ptr(scales), _ptr(scale_exp), nb)


def tgevc_z(T, ldt, S, lds, m, Z, ldz, lam, scales, scale_exp, nb):
    _call("tgevc_z", _ptr(T), ldt, _ptr(S), lds, m, _ptr(Z), ldz, _ptr(lam), _ptr(scales), _ptr(scale_exp), nb)


def pseudospectra_z(U, ldu, m, z, npts, iters, v0, sigma_min, flags, nb):
    _call("pseudospectra_z", _ptr(U), ldu, m, _ptr(z), npts, iters, _ptr(v0), _ptr(sigma_min),
          _ptr(flags), nb)


def pack_cols(Z, heights, offsets, out, src_cols=None):
    """out[offsets[q]:+heights[q]] = Z[:heights[q], src_cols[q]] (CUDA tensors, int64 index tensors)."""
    torch = _torch()
    name = "mstrsm_z_pack_cols" if Z.dtype == torch.complex128 else "mstrsm_d_pack_cols"
    _call(name, _ptr(Z), _ld(Z), heights.shape[0], _ptr(src_cols), _ptr(heights), _ptr(offsets), _ptr(out))


def unpack_cols(inp, heights, offsets, dst_cols, m: int, Z):
    """Z[:heights[q], dst_cols[q]] = inp[offsets[q]:...], rows below set to 0 (CUDA tensors)."""
    torch = _torch()
    name = "mstrsm_z_unpack_cols" if Z.dtype == torch.complex128 else "mstrsm_d_unpack_cols"
    _call(name, _ptr(inp), heights.shape[0], _ptr(heights), _ptr(offsets), _ptr(dst_cols), m, _ptr(Z), _ld(Z))


def dist_shard(m: int, nranks: int, rank: int) -> np.ndarray:
    """Eigenvector indices rank `rank` owns (the library's serpentine block-cyclic map)."""
    lib = load()
    n = int(lib.mstrsm_dist_shard(m, nranks, rank, None))
    if n < 0:
        raise MstrsmError("mstrsm_dist_shard: invalid arguments")
    out = np.empty(max(n, 1), dtype=np.int64)
    lib.mstrsm_dist_shard(m, nranks, rank, out.ctypes.data_as(c_vp))
    return out[:n]


def comm_init(nranks: int, rank: int, group=None):
    """NCCL communicator of the library over `nranks` processes (one per GPU): rank 0 draws the
    id, torch.distributed broadcasts it (nranks = 1 needs no process group)."""
    lib = load()
    _bind_stream(lib)
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        _check(lib.mstrsm_comm_unique_id(uid), "mstrsm_comm_unique_id")
    if nranks > 1:
        import torch
        import torch.distributed as dist
        t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=group)
        uid = ctypes.create_string_buffer(bytes(t.cpu().numpy().tobytes()), 128)
    _check(lib.mstrsm_comm_init(nranks, rank, uid), "mstrsm_comm_init")


def comm_destroy():
    _check(load().mstrsm_comm_destroy(), "mstrsm_comm_destroy")


def trevc_dist(T, m: int, *, nb: int = 64, root: int = 0):
    """TriangEig over every rank of the library communicator: T (column-major CUDA tensor) read on
    `root`; returns (Z, scales, scale_exp) on every rank."""
    torch = _torch()
    dtype = T.dtype if T is not None else torch.complex128
    dev = T.device if T is not None else torch.device("cuda")
    Z = torch.empty((m, m), dtype=dtype, device=dev).t()
    scales = torch.empty(m, dtype=torch.float64, device=dev)
    exps = torch.empty(m, dtype=torch.int32, device=dev)
    name = "trevc_z_dist" if dtype == torch.complex128 else "trevc_d_dist"
    _call(name, _ptr(T), _ld(T) if T is not None else 1, m, _ptr(Z), _ld(Z), _ptr(scales), _ptr(exps), nb, root)
    return Z, scales, exps


def solve_dist(U, shifts, B, m: int, *, safe: bool = True, op: str = "N", nb: int = 64, root: int = 0):
    """This rank's columns of a multi-shift solve over the library communicator (U read on root,
    its upper triangle broadcast); B (m x n_local, column-major CUDA) solved in place.  Returns
    (B, scales, scale_exp)."""
    torch = _torch()
    n = B.shape[1]
    scales = torch.empty(n, dtype=torch.float64, device=B.device)
    exps = torch.empty(n, dtype=torch.int32, device=B.device)
    name = "mstrsm_z_dist" if B.dtype == torch.complex128 else "mstrsm_d_dist"
    _call(name, 1 if safe else 0, 0 if op == "N" else 1, _ptr(U), _ld(U) if U is not None else 1, m, _ptr(shifts), 1,
          _ptr(B), _ld(B), n, _ptr(scales), _ptr(exps), nb, root)
    return B, scales, exps


def mstrsm_workspace_size(m: int, n: int, nb: int, is_complex: bool, safe: bool) -> int:
    return int(load().mstrsm_workspace_size(m, n, nb, int(is_complex), int(safe)))


def mstrsm_d_ex_ws(safe, op, U, ldu, m, shifts, shift_stride, B, ldb, n, row_end, scales, scale_exp, nb,
                   workspace, workspace_bytes):
    arr, p = _row_end(row_end, n)
    _call("mstrsm_d_ex_ws", safe, op, _ptr(U), ldu, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n, p,
          _ptr(scales), _ptr(scale_exp), nb, _ptr(workspace), workspace_bytes)


def mstrsm_z_ex_ws(safe, op, U, ldu, m, shifts, shift_stride, B, ldb, n, row_end, scales, scale_exp, nb,
                   workspace, workspace_bytes):
    arr, p = _row_end(row_end, n)
    _call("mstrsm_z_ex_ws", safe, op, _ptr(U), ldu, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n, p,
          _ptr(scales), _ptr(scale_exp), nb, _ptr(workspace), workspace_bytes)


def mstrsm_d_side(safe, side, uplo, A, lda, m, shifts, shift_stride, B, ldb, n, scales, scale_exp, nb):
    _call("mstrsm_d_side", safe, side, uplo, _ptr(A), lda, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n,
          _ptr(scales), _ptr(scale_exp), nb)


def mstrsm_z_side(safe, side, uplo, A, lda, m, shifts, shift_stride, B, ldb, n, scales, scale_exp, nb):
    _call("mstrsm_z_side", safe, side, uplo, _ptr(A), lda, m, _ptr(shifts), shift_stride, _ptr(B), ldb, n,
          _ptr(scales), _ptr(scale_exp), nb)


def solve_side(A, shifts, B, *, side: str = "L", uplo: str = "U", safe: bool = True, nb: int = 64,
               shift_stride: int = 1):
    """In-place multi-shift solve of the P:58-62 family on column-major CUDA tensors: side "L":
    (A - s_j I) x_j = c_j b_j (B m x n); side "R": x_j^T (A - s_j I) = c_j b_j^T (B n x m, row j);
    uplo "U" / "L".  Returns (B, scales, scale_exp)."""
    torch = _torch()
    m = A.shape[0]
    n = B.shape[1] if side == "L" else B.shape[0]
    cplx = B.dtype == torch.complex128
    scales = torch.empty(n, dtype=torch.float64, device=B.device)
    exps = torch.empty(n, dtype=torch.int32, device=B.device)
    f = mstrsm_z_side if cplx else mstrsm_d_side
    f(1 if safe else 0, 0 if side == "L" else 1, 0 if uplo == "U" else 1, A, _ld(A), m, shifts, shift_stride, B,
      _ld(B), n, scales, exps, nb)
    return B, scales, exps


def spectral_cloud_z(U, ldu, m, z, npts, maxit, tol, v0, sigma, flags, its, nb):
    _call("spectral_cloud_z", _ptr(U), ldu, m, _ptr(z), npts, maxit, float(tol), _ptr(v0), _ptr(sigma),
          _ptr(flags), _ptr(its), nb)


def spectral_window_z(U, ldu, m, x0, x1, nx, y0, y1, ny, maxit, tol, v0, sigma, flags, its, nb):
    _call("spectral_window_z", _ptr(U), ldu, m, float(x0), float(x1), nx, float(y0), float(y1), ny, maxit,
          float(tol), _ptr(v0), _ptr(sigma), _ptr(flags), _ptr(its), nb)


def spectral_portrait_z(U, ldu, m, nx, ny, maxit, tol, v0, sigma, flags, its, window_host, nb):
    _call("spectral_portrait_z", _ptr(U), ldu, m, nx, ny, maxit, float(tol), _ptr(v0), _ptr(sigma),
          _ptr(flags), _ptr(its), window_host, nb)


def mstrsm_status() -> int:
    lib = load()
    _bind_stream(lib)
    return int(lib.mstrsm_status())


def mstrsm_set_sync_status(on: int) -> int:
    return int(load().mstrsm_set_sync_status(1 if on else 0))


def mstrsm_launch_count(reset: int = 0) -> int:
    return int(load().mstrsm_launch_count(reset))


def mstrsm_fp64_peak(ms: float = 50.0):
    lib = load()
    _bind_stream(lib)
    a, b = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib.mstrsm_fp64_peak(ms, ctypes.byref(a), ctypes.byref(b)), "mstrsm_fp64_peak")
    return a.value, b.value


def mstrsm_profile(enable: int):
    lib = load()
    _bind_stream(lib)
    _check(lib.mstrsm_profile(enable), "mstrsm_profile")


def mstrsm_profile_read(kind: int):
    """(total device ms, launches, algorithmic flops) of one kernel kind since mstrsm_profile(1):
    0 = update GEMM, 1 = diagonal-block kernel, 2 = other."""
    lib = load()
    _bind_stream(lib)
    t, c, f = ctypes.c_double(0), ctypes.c_int64(0), ctypes.c_double(0)
    _check(lib.mstrsm_profile_read(kind, ctypes.byref(t), ctypes.byref(c), ctypes.byref(f)),
           "mstrsm_profile_read")
    return t.value, c.value, f.value


def mstrsm_gemm_real_products() -> int:
    """Real DMMA products per complex multiply-add in the update GEMM (3: 3M, 4: four products)."""
    return int(load().mstrsm_gemm_real_products())


def mstrsm_error_string(code: int) -> str:
    return load().mstrsm_error_string(code).decode()


# ------------------------------------------------------------------ convenience wrappers
status = mstrsm_status
launch_count = mstrsm_launch_count
fp64_peak = mstrsm_fp64_peak
gemm_real_products = mstrsm_gemm_real_products


def colmajor(t):
    """Column-major copy of a 2-D tensor (same device / dtype)."""
    return t.t().contiguous().t()


def solve(U, shifts, B, *, safe: bool = True, op: str = "N", nb: int = 64, row_end=None,
          shift_stride: int = 1):
    """In-place multi-shift solve on column-major CUDA tensors; returns (B, scales, scale_exp)."""
    torch = _torch()
    m, n = B.shape
    cplx = B.dtype == torch.complex128
    scales = torch.empty(n, dtype=torch.float64, device=B.device)
    exps = torch.empty(n, dtype=torch.int32, device=B.device)
    f = mstrsm_z_ex if cplx else mstrsm_d_ex
    f(1 if safe else 0, 0 if op == "N" else 1, U, _ld(U), m, shifts, shift_stride, B, _ld(B), n,
      row_end, scales, exps, nb)
    return B, scales, exps


def trevc(T, *, nb: int = 64, cols=None):
    """Triangular eigenvectors of column-major CUDA tensor T; returns (Z, scales, scale_exp)."""
    torch = _torch()
    m = T.shape[0]
    ncols = m if cols is None else len(cols)
    Z = torch.empty((ncols, m), dtype=T.dtype, device=T.device).t()
    scales = torch.empty(ncols, dtype=torch.float64, device=T.device)
    exps = torch.empty(ncols, dtype=torch.int32, device=T.device)
    cplx = T.dtype == torch.complex128
    if cols is None:
        (trevc_z if cplx else trevc_d)(T, _ld(T), m, Z, _ld(Z), scales, exps, nb)
    else:
        (trevc_z_cols if cplx else trevc_d_cols)(T, _ld(T), m, cols, ncols, Z, _ld(Z), scales, exps, nb)
    return Z, scales, exps


def solve_gen(U, V, shifts, B, *, safe: bool = True, nb: int = 64, row_end=None, shift_stride: int = 1):
    """In-place generalized multi-shift solve (U - s_j V) x_j = c_j b_j on column-major CUDA
    tensors (Alg. 7/8); returns (B, scales, scale_exp)."""
    torch = _torch()
    m, n = B.shape
    cplx = B.dtype == torch.complex128
    scales = torch.empty(n, dtype=torch.float64, device=B.device)
    exps = torch.empty(n, dtype=torch.int32, device=B.device)
    f = mstrsm_z_gen if cplx else mstrsm_d_gen
    f(1 if safe else 0, U, _ld(U), V, _ld(V), m, shifts, shift_stride, B, _ld(B), n, row_end, scales, exps, nb)
    return B, scales, exps


def tgevc(T, S, *, nb: int = 64):
    """Eigenvectors of the upper-triangular pencil (T, S) (Alg. 9); returns (Z, lambda, scales,
    scale_exp) as CUDA tensors (Z column-major)."""
    torch = _torch()
    m = T.shape[0]
    Z = torch.empty((m, m), dtype=T.dtype, device=T.device).t()
    lam = torch.empty(m, dtype=T.dtype, device=T.device)
    scales = torch.empty(m, dtype=torch.float64, device=T.device)
    exps = torch.empty(m, dtype=torch.int32, device=T.device)
    f = tgevc_z if T.dtype == torch.complex128 else tgevc_d
    f(T, _ld(T), S, _ld(S), m, Z, _ld(Z), lam, scales, exps, nb)
    return Z, lam, scales, exps


def eig_backtransform_d(Q, ldq, m, Z, ldz, n, cols_host, X, ldx):
    arr, p = _host_i64(cols_host)
    _call("eig_backtransform_d", _ptr(Q), ldq, m, _ptr(Z), ldz, n, p, _ptr(X), ldx)


def eig_backtransform_z(Q, ldq, m, Z, ldz, n, cols_host, X, ldx):
    arr, p = _host_i64(cols_host)
    _call("eig_backtransform_z", _ptr(Q), ldq, m, _ptr(Z), ldz, n, p, _ptr(X), ldx)


def trevc_qz_d(T, ldt, m, Q, ldq, X, ldx, scales, scale_exp, nb):
    _call("trevc_qz_d", _ptr(T), ldt, m, _ptr(Q), ldq, _ptr(X), ldx, _ptr(scales), _ptr(scale_exp), nb)


def trevc_qz_z(T, ldt, m, Q, ldq, X, ldx, scales, scale_exp, nb):
    _call("trevc_qz_z", _ptr(T), ldt, m, _ptr(Q), ldq, _ptr(X), ldx, _ptr(scales), _ptr(scale_exp), nb)


def eig_backtransform(Q, Z, *, cols=None):
    """X = Q Z on column-major CUDA tensors, Z zero below row cols[q] in column q
    (default q: upper triangular); returns X (column-major)."""
    torch = _torch()
    m, n = Z.shape
    X = torch.empty((n, m), dtype=Z.dtype, device=Z.device).t()
    f = eig_backtransform_z if Z.dtype == torch.complex128 else eig_backtransform_d
    f(Q, _ld(Q), m, Z, _ld(Z), n, cols, X, _ld(X))
    return X


def trevc_qz(T, Q, *, nb: int = 64):
    """Eigenvectors of A = Q T Q^H from its Schur pair (TriangEig, then X = Q Z);
    returns (X, scales, scale_exp) as CUDA tensors (X column-major)."""
    torch = _torch()
    m = T.shape[0]
    X = torch.empty((m, m), dtype=T.dtype, device=T.device).t()
    scales = torch.empty(m, dtype=torch.float64, device=T.device)
    exps = torch.empty(m, dtype=torch.int32, device=T.device)
    f = trevc_qz_z if T.dtype == torch.complex128 else trevc_qz_d
    f(T, _ld(T), m, Q, _ld(Q), X, _ld(X), scales, exps, nb)
    return X, scales, exps


def _cloud_out(n, dev):
    torch = _torch()
    return (torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
            torch.empty(n, dtype=torch.int32, device=dev))


def spectral_cloud(U, z, v0, *, maxit: int = 15, tol: float = 1e-10, nb: int = 64):
    """SpectralCloud: sigma_min(U - z_p I) with per-point deflation (R33); returns
    (sigma, flags, its) as CUDA tensors."""
    m, npts = U.shape[0], z.shape[0]
    sigma, flags, its = _cloud_out(npts, U.device)
    spectral_cloud_z(U, _ld(U), m, z, npts, maxit, tol, v0, sigma, flags, its, nb)
    return sigma, flags, its


def spectral_window(U, x0, x1, nx, y0, y1, ny, v0, *, maxit: int = 15, tol: float = 1e-10, nb: int = 64):
    """SpectralWindow over the nx x ny grid (R15 order); returns (sigma, flags, its)."""
    m = U.shape[0]
    sigma, flags, its = _cloud_out(nx * ny, U.device)
    spectral_window_z(U, _ld(U), m, x0, x1, nx, y0, y1, ny, maxit, tol, v0, sigma, flags, its, nb)
    return sigma, flags, its


def spectral_portrait(U, nx, ny, v0, *, maxit: int = 15, tol: float = 1e-10, nb: int = 64):
    """SpectralPortrait: the automatic window of R34; returns (sigma, flags, its, window)."""
    m = U.shape[0]
    sigma, flags, its = _cloud_out(nx * ny, U.device)
    win = (ctypes.c_double * 4)()
    spectral_portrait_z(U, _ld(U), m, nx, ny, maxit, tol, v0, sigma, flags, its, ctypes.cast(win, c_vp), nb)
    return sigma, flags, its, tuple(win)


def pseudospectra(U, z, v0, *, iters: int = 15, nb: int = 64):
    """sigma_min(U - z_p I) for all points; returns (sigma, flags)."""
    torch = _torch()
    m = U.shape[0]
    npts = z.shape[0]
    sigma = torch.empty(npts, dtype=torch.float64, device=U.device)
    flags = torch.empty(npts, dtype=torch.int32, device=U.device)
    pseudospectra_z(U, _ld(U), m, z, npts, iters, v0, sigma, flags, nb)
    return sigma, flags

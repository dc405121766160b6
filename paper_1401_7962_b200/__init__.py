"""paper_1401_7962_b200 — B200-native Gauss–Jordan inversion (arxiv 1401.7962).

Thin Python binding over the C-ABI library ``libgjinv.so`` (``include/gjinv.h``).
Argument marshalling only: torch supplies device memory and the current CUDA stream;
every step of the method runs in the library's sm_100a kernels.  There is no CPU
fallback: if the library cannot be loaded, importing this package raises.

Entry points mirror the C names: :func:`invert_batched`, :func:`invert_batched_full`,
:func:`invert`, :func:`det`, :func:`invert_batched_host`.
"""
from __future__ import annotations

import ctypes
import os
from collections import namedtuple
from typing import Optional

from ._build import LIB as _LIB_PATH

__all__ = ["invert_batched", "invert_batched_full", "invert_batched_pivoting", "solve_batched", "solve", "invert",
           "det", "invert_batched_host", "GJError", "lib", "library_path",
           "TOL_DEFAULT", "Result"]

TOL_DEFAULT = -1.0
GJ_F32, GJ_F64 = 0, 1


class GJError(RuntimeError):
    pass


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"libgjinv.so not built at {_LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.gj_invert_batched.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    L.gj_invert_batched.restype = i32
    L.gj_invert_batched_full.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    L.gj_invert_batched_full.restype = i32
    L.gj_invert_batched_pivoting.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, dbl, i32, vp]
    L.gj_invert_batched_pivoting.restype = i32
    L.gj_solve_batched.argtypes = [i32, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    L.gj_solve_batched.restype = i32
    L.gj_solve.argtypes = [i32, i32, i32, vp, i64, vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
    L.gj_solve.restype = i32
    L.gj_solve_workspace_size.argtypes = [i32, i32, i32]
    L.gj_solve_workspace_size.restype = ctypes.c_size_t
    L.gj_det.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
    L.gj_det.restype = i32
    L.gj_invert.argtypes = [i32, i32, vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
    L.gj_invert.restype = i32
    L.gj_workspace_size.argtypes = [i32, i32, i64, i32]
    L.gj_workspace_size.restype = ctypes.c_size_t
    L.gj_invert_batched_host.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, i64]
    L.gj_invert_batched_host.restype = i32
    L.gj_host_release.restype = i32
    ub = ctypes.POINTER(ctypes.c_ubyte)
    L.gj_dist_get_unique_id.argtypes = [ub]
    L.gj_dist_get_unique_id.restype = i32
    L.gj_dist_init.argtypes = [i32, i32, ub, i32, ctypes.POINTER(ctypes.c_void_p)]
    L.gj_dist_init.restype = i32
    L.gj_invert_dist.argtypes = [vp, i32, vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp]
    L.gj_invert_dist.restype = i32
    L.gj_dist_finalize.argtypes = [vp]
    L.gj_dist_finalize.restype = i32
    L.gj_status_string.argtypes = [i32]
    L.gj_status_string.restype = ctypes.c_char_p
    L.gj_version.restype = ctypes.c_char_p
    return L


lib = _load()
library_path = _LIB_PATH

Result = namedtuple("Result", ["inverse", "logabsdet", "sign", "det", "ipiv", "info"])
FullResult = namedtuple("FullResult", ["inverse", "logabsdet", "sign", "det", "ipiv", "jpiv", "info"])


def _check(st: int):
    if st != 0:
        raise GJError(lib.gj_status_string(st).decode())


def _torch():
    import torch
    return torch


def _dt(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return GJ_F32
    if t.dtype == torch.float64:
        return GJ_F64
    raise TypeError(f"unsupported dtype {t.dtype} (float32 / float64)")


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _check_out(out, shape, dtype, device, name="out", contiguous=True, unit_col=False):
    """A caller-provided output must match what the library writes (no silent
    out-of-bounds writes through a raw pointer)."""
    if out is None:
        return
    if tuple(out.shape) != tuple(shape) or out.dtype != dtype or out.device != device:
        raise ValueError(f"{name} must be {dtype} {tuple(shape)} on {device}, got {out.dtype} "
                         f"{tuple(out.shape)} on {out.device}")
    if contiguous and not out.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if unit_col and out.dim() == 2 and out.stride(1) != 1:
        raise ValueError(f"{name} must have unit column stride")


def _check_square_batch(A, what="A"):
    if not A.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if A.dim() != 3 or A.shape[1] != A.shape[2]:
        raise ValueError(f"{what} must be [B, n, n]")
    if not A.is_contiguous():
        raise ValueError(f"{what} must be contiguous")


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def invert_batched(A, tol: Optional[float] = None, *, out=None, inverse: bool = True, ipiv: bool = True,
                   logabsdet: bool = True, sign: bool = True, det: bool = True, info: bool = True,
                   stream=None) -> Result:
    """Invert a batch ``A`` ([B, n, n] or [n, n], float32/float64, CUDA, contiguous) with
    ``gj_invert_batched``.  ``tol``: relative zero threshold (None → n·eps).  ``out`` may be
    ``A`` itself for an in-place inversion.  Unrequested outputs are None."""
    torch = _torch()
    if not A.is_cuda:
        raise ValueError("A must be a CUDA tensor (use invert_batched_host for host buffers)")
    squeeze = A.dim() == 2
    if squeeze:
        A = A.unsqueeze(0)
    if A.dim() != 3 or A.shape[1] != A.shape[2]:
        raise ValueError("A must be [B, n, n]")
    if not A.is_contiguous():
        raise ValueError("A must be contiguous")
    B, n = A.shape[0], A.shape[1]
    dev = A.device
    X = None
    if inverse:
        if out is not None and out.dim() == 2 and squeeze:
            out = out.unsqueeze(0)
        _check_out(out, A.shape, A.dtype, dev)
        X = out if out is not None else torch.empty_like(A)
    o_ipiv = torch.empty((B, n), dtype=torch.int32, device=dev) if ipiv else None
    o_lg = torch.empty((B,), dtype=torch.float64, device=dev) if logabsdet else None
    o_sg = torch.empty((B,), dtype=torch.int8, device=dev) if sign else None
    o_det = torch.empty((B,), dtype=A.dtype, device=dev) if det else None
    o_info = torch.empty((B,), dtype=torch.int32, device=dev) if info else None
    with torch.cuda.device(dev):
        st = lib.gj_invert_batched(_dt(A), n, B, A.data_ptr(), _ptr(X), _ptr(o_ipiv), _ptr(o_lg), _ptr(o_sg),
                                   _ptr(o_det), _ptr(o_info), TOL_DEFAULT if tol is None else float(tol),
                                   _stream_ptr(stream))
    _check(st)
    if squeeze:
        sq = lambda t: None if t is None else t[0]
        return Result(sq(X), sq(o_lg), sq(o_sg), sq(o_det), sq(o_ipiv), sq(o_info))
    return Result(X, o_lg, o_sg, o_det, o_ipiv, o_info)


SolveResult = namedtuple("SolveResult", ["X", "logabsdet", "sign", "ipiv", "info"])


def solve_batched(A, B, tol: Optional[float] = None, *, out=None, ipiv: bool = True, stream=None) -> "SolveResult":
    """``gj_solve_batched``: X = A^-1 B by Gauss–Jordan on [A | B] (n, nrhs ≤ 32).
    A [batch, n, n], B [batch, n, nrhs] (or [n, n], [n, nrhs]); ``out`` may be B.
    ``ipiv=False`` requests no pivot sequence (fp32 n = 32 then runs the two-pass K1f
    scheme; the result's ipiv is None)."""
    torch = _torch()
    if not (A.is_cuda and B.is_cuda):
        raise ValueError("A and B must be CUDA tensors")
    squeeze = A.dim() == 2
    if squeeze:
        A, B = A.unsqueeze(0), B.unsqueeze(0)
    if A.dim() != 3 or A.shape[1] != A.shape[2] or B.dim() != 3 or B.shape[:2] != A.shape[:2]:
        raise ValueError("A must be [batch, n, n] and B [batch, n, nrhs]")
    if not (A.is_contiguous() and B.is_contiguous()) or A.dtype != B.dtype:
        raise ValueError("A and B must be contiguous and of one dtype")
    bt, n, m = A.shape[0], A.shape[1], B.shape[2]
    dev = A.device
    if B.device != dev:
        raise ValueError("A and B must be on one device")
    if out is not None and out.dim() == 2 and squeeze:
        out = out.unsqueeze(0)
    _check_out(out, B.shape, B.dtype, dev)
    X = out if out is not None else torch.empty_like(B)
    o_ipiv = torch.empty((bt, n), dtype=torch.int32, device=dev) if ipiv else None
    o_lg = torch.empty((bt,), dtype=torch.float64, device=dev)
    o_sg = torch.empty((bt,), dtype=torch.int8, device=dev)
    o_info = torch.empty((bt,), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = lib.gj_solve_batched(_dt(A), n, m, bt, A.data_ptr(), B.data_ptr(), X.data_ptr(), _ptr(o_ipiv),
                                  o_lg.data_ptr(), o_sg.data_ptr(), o_info.data_ptr(),
                                  TOL_DEFAULT if tol is None else float(tol), _stream_ptr(stream))
    _check(st)
    if squeeze:
        return SolveResult(X[0], o_lg[0], o_sg[0], None if o_ipiv is None else o_ipiv[0], o_info[0])
    return SolveResult(X, o_lg, o_sg, o_ipiv, o_info)


def solve(A, B, tol: Optional[float] = None, *, out=None, stream=None) -> "SolveResult":
    """``gj_solve``: one system X = A^-1 B of any order (strided rows allowed on the large
    path; fp64 beyond n, nrhs <= 32)."""
    torch = _torch()
    if A.dim() != 2 or A.shape[0] != A.shape[1] or B.dim() != 2 or B.shape[0] != A.shape[0]:
        raise ValueError("A must be [n, n] and B [n, nrhs]")
    if A.stride(1) != 1 or B.stride(1) != 1 or A.dtype != B.dtype:
        raise ValueError("unit column stride and one dtype required")
    n, m = A.shape[0], B.shape[1]
    dev = A.device
    if not (A.is_cuda and B.is_cuda) or B.device != dev:
        raise ValueError("A and B must be CUDA tensors on one device")
    _check_out(out, (n, m), A.dtype, dev, contiguous=False, unit_col=True)
    X = out if out is not None else torch.empty((n, m), dtype=A.dtype, device=dev)
    o_ipiv = torch.empty((n,), dtype=torch.int32, device=dev)
    o_lg = torch.empty((1,), dtype=torch.float64, device=dev)
    o_sg = torch.empty((1,), dtype=torch.int8, device=dev)
    o_info = torch.empty((1,), dtype=torch.int32, device=dev)
    ws_bytes = lib.gj_solve_workspace_size(_dt(A), n, m)
    ws = torch.empty((max(ws_bytes, 1),), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = lib.gj_solve(_dt(A), n, m, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), X.data_ptr(),
                          X.stride(0), o_ipiv.data_ptr(), o_lg.data_ptr(), o_sg.data_ptr(), o_info.data_ptr(),
                          TOL_DEFAULT if tol is None else float(tol), ws.data_ptr(), ws_bytes, _stream_ptr(stream))
    _check(st)
    return SolveResult(X, o_lg[0], o_sg[0], o_ipiv, o_info[0])


PIVOTING = {"none": 0, "partial": 1, "full": 2}


def invert_batched_pivoting(A, strategy: str = "full", tol: Optional[float] = None, *, out=None,
                            inverse: bool = True, pivots: bool = True, stream=None) -> "FullResult":
    """``gj_invert_batched_pivoting`` (n ≤ 32): the K6 kernel with ``strategy`` "none"
    (pivot a_kk, Eqs. (3)–(10)), "partial" (the listing's row search) or "full"
    (Obs. 2–3); as :func:`invert_batched` plus ``jpiv``, the column swap sequence.
    ``pivots=False`` requests neither ipiv nor jpiv (their fields are None; full pivoting
    at fp32 n = 32 then runs the two-pass K6f scheme)."""
    torch = _torch()
    if not A.is_cuda:
        raise ValueError("A must be a CUDA tensor")
    squeeze = A.dim() == 2
    if squeeze:
        A = A.unsqueeze(0)
    if A.dim() != 3 or A.shape[1] != A.shape[2] or not A.is_contiguous():
        raise ValueError("A must be a contiguous [B, n, n]")
    B, n = A.shape[0], A.shape[1]
    dev = A.device
    if inverse and out is not None and out.dim() == 2 and squeeze:
        out = out.unsqueeze(0)
    if inverse:
        _check_out(out, A.shape, A.dtype, dev)
    X = (out if out is not None else torch.empty_like(A)) if inverse else None
    o_ipiv = torch.empty((B, n), dtype=torch.int32, device=dev) if pivots else None
    o_jpiv = torch.empty((B, n), dtype=torch.int32, device=dev) if pivots else None
    o_lg = torch.empty((B,), dtype=torch.float64, device=dev)
    o_sg = torch.empty((B,), dtype=torch.int8, device=dev)
    o_det = torch.empty((B,), dtype=A.dtype, device=dev)
    o_info = torch.empty((B,), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        st = lib.gj_invert_batched_pivoting(_dt(A), n, B, A.data_ptr(), _ptr(X), _ptr(o_ipiv),
                                            _ptr(o_jpiv), o_lg.data_ptr(), o_sg.data_ptr(), o_det.data_ptr(),
                                            o_info.data_ptr(), TOL_DEFAULT if tol is None else float(tol),
                                            PIVOTING[strategy], _stream_ptr(stream))
    _check(st)
    if squeeze:
        sq = lambda t: None if t is None else t[0]
        return FullResult(sq(X), o_lg[0], o_sg[0], o_det[0], sq(o_ipiv), sq(o_jpiv), o_info[0])
    return FullResult(X, o_lg, o_sg, o_det, o_ipiv, o_jpiv, o_info)


def invert_batched_full(A, tol: Optional[float] = None, *, out=None, inverse: bool = True,
                        pivots: bool = True, stream=None) -> "FullResult":
    """Full pivoting (``gj_invert_batched_full``, Obs. 2–3; n ≤ 32): as
    :func:`invert_batched` plus ``jpiv``, the 1-based column swap sequence."""
    return invert_batched_pivoting(A, "full", tol, out=out, inverse=inverse, pivots=pivots, stream=stream)


def det(A, tol: Optional[float] = None, *, ipiv: bool = True, stream=None) -> Result:
    """Determinants only (``gj_det``): logabsdet, sign, det, ipiv, info; inverse is None.
    ``ipiv=False`` requests no pivot sequence (its field is then None)."""
    torch = _torch()
    squeeze = A.dim() == 2
    if squeeze:
        A = A.unsqueeze(0)
    _check_square_batch(A)
    B, n = A.shape[0], A.shape[1]
    dev = A.device
    o_ipiv = torch.empty((B, n), dtype=torch.int32, device=dev) if ipiv else None
    o_lg = torch.empty((B,), dtype=torch.float64, device=dev)
    o_sg = torch.empty((B,), dtype=torch.int8, device=dev)
    o_det = torch.empty((B,), dtype=A.dtype, device=dev)
    o_info = torch.empty((B,), dtype=torch.int32, device=dev)
    ws_bytes = lib.gj_workspace_size(_dt(A), n, B, 2)
    ws = torch.empty((max(ws_bytes, 1),), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = lib.gj_det(_dt(A), n, B, A.data_ptr(), o_lg.data_ptr(), o_sg.data_ptr(), o_det.data_ptr(),
                        _ptr(o_ipiv), o_info.data_ptr(), TOL_DEFAULT if tol is None else float(tol),
                        ws.data_ptr(), ws_bytes, _stream_ptr(stream))
    _check(st)
    if squeeze:
        return Result(None, o_lg[0], o_sg[0], o_det[0], None if o_ipiv is None else o_ipiv[0], o_info[0])
    return Result(None, o_lg, o_sg, o_det, o_ipiv, o_info)


def invert(A, tol: Optional[float] = None, *, out=None, stream=None) -> Result:
    """One matrix of any order (``gj_invert``); strided rows are allowed."""
    torch = _torch()
    if A.dim() != 2 or A.shape[0] != A.shape[1] or A.stride(1) != 1:
        raise ValueError("A must be [n, n] with unit column stride")
    if not A.is_cuda:
        raise ValueError("A must be a CUDA tensor")
    n = A.shape[0]
    dev = A.device
    _check_out(out, (n, n), A.dtype, dev, contiguous=False, unit_col=True)
    X = out if out is not None else torch.empty((n, n), dtype=A.dtype, device=dev)
    o_ipiv = torch.empty((n,), dtype=torch.int32, device=dev)
    o_lg = torch.empty((1,), dtype=torch.float64, device=dev)
    o_sg = torch.empty((1,), dtype=torch.int8, device=dev)
    o_info = torch.empty((1,), dtype=torch.int32, device=dev)
    ws_bytes = lib.gj_workspace_size(_dt(A), n, 1, 1)
    ws = torch.empty((max(ws_bytes, 1),), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = lib.gj_invert(_dt(A), n, A.data_ptr(), A.stride(0), X.data_ptr(), X.stride(0), o_ipiv.data_ptr(),
                           o_lg.data_ptr(), o_sg.data_ptr(), o_info.data_ptr(),
                           TOL_DEFAULT if tol is None else float(tol), ws.data_ptr(), ws_bytes,
                           _stream_ptr(stream))
    _check(st)
    return Result(X, o_lg[0], o_sg[0], None, o_ipiv, o_info[0])


def invert_batched_host(A, tol: Optional[float] = None, *, out=None, ipiv=None, logabsdet=None, sign=None,
                        det=None, info=None, chunk: int = 0):
    """``gj_invert_batched_host`` on host (CPU) tensors/arrays; synchronous.  ``out`` and the
    optional side outputs are caller-provided host buffers (pinned → overlapped copies)."""
    def ptr(t):
        if t is None:
            return None
        if hasattr(t, "data_ptr"):
            return t.data_ptr()
        return t.ctypes.data
    torch = _torch()
    import numpy as np
    if isinstance(A, torch.Tensor):
        if A.is_cuda:
            raise ValueError("invert_batched_host takes host tensors / arrays")
        dt = _dt(A)
        fdt = A.dtype
        contig = lambda t: t.is_contiguous()
        same = lambda t, dtp: isinstance(t, torch.Tensor) and not t.is_cuda and t.dtype == dtp
        tdt = {"i32": torch.int32, "f64": torch.float64, "i8": torch.int8}
    else:
        A = np.asarray(A)
        if A.dtype == np.float32:
            dt = GJ_F32
        elif A.dtype == np.float64:
            dt = GJ_F64
        else:
            raise TypeError(f"unsupported dtype {A.dtype} (float32 / float64)")
        fdt = A.dtype
        contig = lambda t: t.flags["C_CONTIGUOUS"]
        same = lambda t, dtp: isinstance(t, np.ndarray) and t.dtype == dtp
        tdt = {"i32": np.int32, "f64": np.float64, "i8": np.int8}
    if A.ndim != 3 or A.shape[1] != A.shape[2] or not contig(A):
        raise ValueError("A must be a C-contiguous [B, n, n] host array")
    B, n = A.shape[0], A.shape[1]
    for t, name, shape, dtp in ((out, "out", (B, n, n), fdt), (ipiv, "ipiv", (B, n), tdt["i32"]),
                                (logabsdet, "logabsdet", (B,), tdt["f64"]), (sign, "sign", (B,), tdt["i8"]),
                                (det, "det", (B,), fdt), (info, "info", (B,), tdt["i32"])):
        if t is None:
            continue
        if not same(t, dtp) or tuple(t.shape) != shape or not contig(t):
            raise ValueError(f"{name} must be a C-contiguous host {dtp} {shape}")
    st = lib.gj_invert_batched_host(dt, n, B, ptr(A), ptr(out), ptr(ipiv), ptr(logabsdet), ptr(sign), ptr(det),
                                    ptr(info), TOL_DEFAULT if tol is None else float(tol), int(chunk))
    _check(st)
    return out


def host_release() -> None:
    """``gj_host_release``: free the staging buffers and streams kept by
    :func:`invert_batched_host` (all devices)."""
    _check(lib.gj_host_release())


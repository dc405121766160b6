"""CPU oracle for Gauss–Jordan inversion — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1401_7962_b200``) never imports it, and the two share no code: the only
module both sides use is ``synth`` (seeded input generators, none of the method's
arithmetic).

* :func:`invert` / :func:`invert_batched` — the textbook long-double Gauss–Jordan on
  the augmented system [A | I] (``oracle/gj_oracle.c``; §2 Eqs. (1)–(2),
  (13)–(15), Obs. 2–3, listing L150–L177).  Every step cites its passage there.
* :mod:`oracle.exact` — exact rational brute force (Laplace cofactor determinant,
  adjugate inverse) for n ≤ 6.

Pins (``tests/test_oracle_*.py``, ``-m "not gpu"``) tie this oracle to the paper's
worked matrix, brute force, closed forms (Hadamard, permutation,
second-difference, Hilbert), the LAPACK getrf special case and invariants.  No function
here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gj_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile ``gj_oracle.c`` (gcc, OpenMP) into ``oracle/liboracle.so``."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        lp = ctypes.POINTER(ctypes.c_int64)
        lib.gjo_invert_batched.argtypes = [ctypes.c_int, ctypes.c_int64, dp, ctypes.c_double, ctypes.c_int,
                                           dp, ip, dp, dp, ip, dp, ip, dp, dp, ctypes.c_int]
        lib.gjo_invert_batched.restype = ctypes.c_int
        lib.gjo_invert.argtypes = [ctypes.c_int, dp, ctypes.c_double, ctypes.c_int,
                                   dp, ip, dp, dp, ip, dp, ip, dp, dp, ctypes.c_int]
        lib.gjo_invert.restype = ctypes.c_int
        lib.gjo_steps.argtypes = [ctypes.c_int, dp, ctypes.c_int, ctypes.c_int, dp]
        lib.gjo_steps.restype = ctypes.c_int
        lib.gjo_residual_rows.argtypes = [ctypes.c_int, dp, dp, lp, ctypes.c_int64, ctypes.c_int]
        lib.gjo_residual_rows.restype = ctypes.c_double
        lib.gjo_residual_batched.argtypes = [ctypes.c_int, ctypes.c_int64, dp, dp, dp, ctypes.c_int]
        lib.gjo_residual_batched.restype = ctypes.c_int
        lib.gjo_invert_full_batched.argtypes = [ctypes.c_int, ctypes.c_int64, dp, ctypes.c_double, dp, ip, ip, dp,
                                                dp, ip, dp, ip, dp, dp, ctypes.c_int]
        lib.gjo_invert_full_batched.restype = ctypes.c_int
        lib.gjo_solve_batched.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, dp, dp, ctypes.c_double, dp,
                                          ip, dp, ip, ip, dp, ctypes.c_int]
        lib.gjo_solve_batched.restype = ctypes.c_int
        lib.gjo_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


STRATEGY = {"none": 0, "partial": 1}


@dataclass
class OracleResult:
    """Per-item oracle outputs (batched arrays; a single matrix has batch 1)."""
    inverse: np.ndarray      # [B, n, n] float64 (NaN for singular items)
    ipiv: np.ndarray         # [B, n] int32, LAPACK-style 1-based swap sequence (reading G13)
    pivots: np.ndarray       # [B, n] float64, a_kk^{k-1} after the swap (Eq. (13) factors)
    logabsdet: np.ndarray    # [B] float64
    sign: np.ndarray         # [B] int32 (-1, 0, +1)
    det: np.ndarray          # [B] float64
    info: np.ndarray         # [B] int32, 0 or first failing step (1-based)
    gap: np.ndarray          # [B, n] (c1 - c2) / c1 of the step-k candidates (rule R3)
    cmax_rel: np.ndarray     # [B, n] c1 / max|a_ij| (rule R7)
    jpiv: np.ndarray = None  # [B, n] int32 column swap sequence (full pivoting only)


def threads() -> int:
    return int(_load().gjo_max_threads())


def invert_batched(A, tol: float = 0.0, strategy: str = "partial", nthreads: int = 0) -> OracleResult:
    """Textbook GJ on [A | I] for every item of ``A`` ([B, n, n] or [n, n]; fp32 inputs
    are widened exactly to fp64 first).  ``tol`` is the relative zero threshold: item b
    is singular at the first step whose largest candidate is ≤ tol · max|A_b| (G1)."""
    lib = _load()
    A = np.asarray(A)
    if A.ndim == 2:
        A = A[None]
    if not np.all(np.isfinite(A)):
        raise ValueError("oracle rejects non-finite inputs (reading G20)")
    A = np.ascontiguousarray(A, dtype=np.float64)
    B, n, n2 = A.shape
    assert n == n2
    out = OracleResult(
        inverse=np.empty((B, n, n)), ipiv=np.zeros((B, n), np.int32), pivots=np.zeros((B, n)),
        logabsdet=np.empty(B), sign=np.zeros(B, np.int32), det=np.empty(B), info=np.zeros(B, np.int32),
        gap=np.empty((B, n)), cmax_rel=np.empty((B, n)))
    dp, ip = ctypes.c_double, ctypes.c_int32
    rc = lib.gjo_invert_batched(n, B, _p(A, dp), float(tol), STRATEGY[strategy],
                                _p(out.inverse, dp), _p(out.ipiv, ip), _p(out.pivots, dp),
                                _p(out.logabsdet, dp), _p(out.sign, ip), _p(out.det, dp), _p(out.info, ip),
                                _p(out.gap, dp), _p(out.cmax_rel, dp), int(nthreads))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


def invert(A, tol: float = 0.0, strategy: str = "partial", nthreads: int = 0) -> OracleResult:
    """One (possibly large) matrix; OpenMP over the rows of each elimination step."""
    lib = _load()
    A = np.ascontiguousarray(np.asarray(A), dtype=np.float64)
    n = A.shape[0]
    if not np.all(np.isfinite(A)):
        raise ValueError("oracle rejects non-finite inputs (reading G20)")
    out = OracleResult(
        inverse=np.empty((1, n, n)), ipiv=np.zeros((1, n), np.int32), pivots=np.zeros((1, n)),
        logabsdet=np.empty(1), sign=np.zeros(1, np.int32), det=np.empty(1), info=np.zeros(1, np.int32),
        gap=np.empty((1, n)), cmax_rel=np.empty((1, n)))
    dp, ip = ctypes.c_double, ctypes.c_int32
    nt = int(nthreads) if nthreads else threads()
    rc = lib.gjo_invert(n, _p(A, dp), float(tol), STRATEGY[strategy],
                        _p(out.inverse, dp), _p(out.ipiv, ip), _p(out.pivots, dp),
                        _p(out.logabsdet, dp), _p(out.sign, ip), _p(out.det, dp), _p(out.info, ip),
                        _p(out.gap, dp), _p(out.cmax_rel, dp), nt)
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


def invert_full_batched(A, tol: float = 0.0, nthreads: int = 0) -> OracleResult:
    """Full pivoting (Obs. 2–3; ``gjo_invert_full`` F1–F3): the pivot of
    step k is the first maximum of |a_ij| over i, j = k..n in row-major scan of the
    physically swapped array (reading G23); rows and columns are swapped and the column
    swaps undone at the end.  ``ipiv`` / ``jpiv`` are the 1-based row / column swap
    sequences; ``gap`` is over all candidates of a step."""
    lib = _load()
    A = np.asarray(A)
    if A.ndim == 2:
        A = A[None]
    if not np.all(np.isfinite(A)):
        raise ValueError("oracle rejects non-finite inputs (reading G20)")
    A = np.ascontiguousarray(A, dtype=np.float64)
    B, n, _ = A.shape
    out = OracleResult(
        inverse=np.empty((B, n, n)), ipiv=np.zeros((B, n), np.int32), pivots=np.zeros((B, n)),
        logabsdet=np.empty(B), sign=np.zeros(B, np.int32), det=np.empty(B), info=np.zeros(B, np.int32),
        gap=np.empty((B, n)), cmax_rel=np.empty((B, n)), jpiv=np.zeros((B, n), np.int32))
    dp, ip = ctypes.c_double, ctypes.c_int32
    rc = lib.gjo_invert_full_batched(n, B, _p(A, dp), float(tol), _p(out.inverse, dp), _p(out.ipiv, ip),
                                     _p(out.jpiv, ip), _p(out.pivots, dp), _p(out.logabsdet, dp),
                                     _p(out.sign, ip), _p(out.det, dp), _p(out.info, ip), _p(out.gap, dp),
                                     _p(out.cmax_rel, dp), int(nthreads))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


@dataclass
class SolveResult:
    X: np.ndarray            # [B, n, m] float64 (NaN for failed items)
    ipiv: np.ndarray         # [B, n] int32
    logabsdet: np.ndarray    # [B]
    sign: np.ndarray         # [B] int32
    info: np.ndarray         # [B] int32
    gap: np.ndarray          # [B, n]


def solve_batched(A, B, tol: float = 0.0, nthreads: int = 0) -> SolveResult:
    """Gauss–Jordan on [A | B] (``gjo_solve``; Eqs. (14)–(15) with B in place of I, the
    listing's partial pivoting): X = A^-1 B per item.  A [Bt, n, n], B [Bt, n, m]."""
    lib = _load()
    A = np.asarray(A)
    Bm = np.asarray(B)
    if A.ndim == 2:
        A, Bm = A[None], Bm[None]
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(Bm))):
        raise ValueError("oracle rejects non-finite inputs (reading G20)")
    A = np.ascontiguousarray(A, dtype=np.float64)
    Bm = np.ascontiguousarray(Bm, dtype=np.float64)
    Bt, n, _ = A.shape
    m = Bm.shape[2]
    out = SolveResult(X=np.empty((Bt, n, m)), ipiv=np.zeros((Bt, n), np.int32), logabsdet=np.empty(Bt),
                      sign=np.zeros(Bt, np.int32), info=np.zeros(Bt, np.int32), gap=np.empty((Bt, n)))
    dp, ip = ctypes.c_double, ctypes.c_int32
    rc = lib.gjo_solve_batched(n, m, Bt, _p(A, dp), _p(Bm, dp), float(tol), _p(out.X, dp), _p(out.ipiv, ip),
                               _p(out.logabsdet, dp), _p(out.sign, ip), _p(out.info, ip), _p(out.gap, dp),
                               int(nthreads))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


def steps(A, nsteps: int, strategy: str = "partial") -> np.ndarray:
    """The working array [A^k | D^k] (n × 2n) after ``nsteps`` steps (Eqs. (3)–(10)/(14)–(15))."""
    lib = _load()
    A = np.ascontiguousarray(np.asarray(A), dtype=np.float64)
    n = A.shape[0]
    M = np.empty((n, 2 * n))
    lib.gjo_steps(n, _p(A, ctypes.c_double), int(nsteps), STRATEGY[strategy], _p(M, ctypes.c_double))
    return M


def residual(A, X, rows=None, nthreads: int = 0) -> float:
    """max |A·X − I| over the given rows (all rows if None), long-double accumulation (G17)."""
    lib = _load()
    A = np.ascontiguousarray(np.asarray(A), dtype=np.float64)
    X = np.ascontiguousarray(np.asarray(X), dtype=np.float64)
    n = A.shape[0]
    if rows is None:
        return float(lib.gjo_residual_rows(n, _p(A, ctypes.c_double), _p(X, ctypes.c_double), None, 0, int(nthreads)))
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    return float(lib.gjo_residual_rows(n, _p(A, ctypes.c_double), _p(X, ctypes.c_double),
                                       _p(r, ctypes.c_int64), len(r), int(nthreads)))


def residual_batched(A, X, nthreads: int = 0) -> np.ndarray:
    """Per item max |A_b·X_b − I| (long-double accumulation)."""
    lib = _load()
    A = np.ascontiguousarray(np.asarray(A), dtype=np.float64)
    X = np.ascontiguousarray(np.asarray(X), dtype=np.float64)
    B, n, _ = A.shape
    out = np.empty(B)
    lib.gjo_residual_batched(n, B, _p(A, ctypes.c_double), _p(X, ctypes.c_double), _p(out, ctypes.c_double),
                             int(nthreads))
    return out


def kappa_inf(A, Ainv) -> np.ndarray:
    """κ∞ = ‖A‖∞ · ‖A⁻¹‖∞ per item, from the oracle's own inverse (rules R1–R5)."""
    A = np.asarray(A, dtype=np.float64)
    Ainv = np.asarray(Ainv, dtype=np.float64)
    if A.ndim == 2:
        A, Ainv = A[None], Ainv[None]
    return np.abs(A).sum(axis=2).max(axis=1) * np.abs(Ainv).sum(axis=2).max(axis=1)

"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no elimination, pivoting,
determinants or inverses): it only draws matrices.  It is the one module both
``oracle/`` (via the tests) and ``paper_1401_7962_b200`` (via bench.py / smoke) use.

Generator = numpy ``default_rng(seed)`` (PCG64).  Recipes follow BASELINE.json
``configs`` C1..C5 with the readings written in DESIGN.md §3:

* C1  seed 0: 4096 × 16×16 fp64, uniform[-1,1] + 16·I; item 0 = blockdiag(P3, I13)
      where P3 = [[1,1,1],[1,2,3],[1,3,6]] is the paper's default matrix.
* C2  seed 1: 1,048,576 × 32×32 fp32 N(0,1), drawn in fixed 65,536-item chunks.
* C3  seed 2: 262,144 × 64×64 fp64 = row-permuted L·diag(u) (L unit-lower, N(0, 0.5)
      strictly-lower; u ~ U[0.5, 2]), then ⌊1%⌋ items get a duplicated row (singular).
* C4  seed 3: 8192×8192 fp64 N(0,1)/√n.      C5  seed 4: 32768×32768 fp64 N(0,1)/√n.
* Exact companions: Sylvester–Hadamard P·H·D (seed 5), permutation matrices, signed
  permutation × power-of-two diagonal, second-difference tridiag(−1,2,−1), Hilbert.
"""
from __future__ import annotations

import itertools
from typing import Iterator, Optional

import numpy as np

PAPER_MATRIX = [[1.0, 1.0, 1.0], [1.0, 2.0, 3.0], [1.0, 3.0, 6.0]]  # PAPER.md L89–L92 ("matrice implicita")

C2_CHUNK = 65536
C3_CHUNK = 8192

CONFIGS = {
    # name: (batch, n, dtype, seed)
    "C1": (4096, 16, np.float64, 0),
    "C2": (1048576, 32, np.float32, 1),
    "C3": (262144, 64, np.float64, 2),
    "C4": (1, 8192, np.float64, 3),
    "C5": (1, 32768, np.float64, 4),
}

# Relative zero thresholds stated per config (reading G1): C3 states 1e-10; the others use
# the library default n·eps(dtype).
C3_TOL = 1e-10


def paper_matrix(dtype=np.float64) -> np.ndarray:
    return np.array(PAPER_MATRIX, dtype=dtype)


def gen_c1(batch: int = 4096, seed: int = 0) -> np.ndarray:
    """BASELINE.json configs[0] (reading G14: item 0 = blockdiag(P3, I13))."""
    n = 16
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (batch, n, n)) + 16.0 * np.eye(n)
    A[0] = np.eye(n)
    A[0, :3, :3] = PAPER_MATRIX
    return np.ascontiguousarray(A)


def gen_c2(batch: int = 1048576, seed: int = 1, out: Optional[np.ndarray] = None,
           chunk: int = C2_CHUNK) -> np.ndarray:
    """BASELINE.json configs[1]: i.i.d. N(0,1) fp32, chunked in order from one generator.
    A smaller ``batch`` yields exactly the prefix of the full-size stream."""
    n = 32
    rng = np.random.default_rng(seed)
    if out is None:
        out = np.empty((batch, n, n), dtype=np.float32)
    for s in range(0, batch, chunk):
        e = min(batch, s + chunk)
        out[s:e] = rng.standard_normal((e - s, n, n), dtype=np.float32)
    return out


def gen_c2_shard(lo: int, hi: int, seed: int = 1, chunk: int = C2_CHUNK) -> np.ndarray:
    """Items [lo, hi) of the C2 stream (the same values gen_c2 gives there): the chunks
    before ``lo`` are drawn and dropped, so a rank's contiguous shard of the seed-1 batch
    is reproduced without holding the whole batch."""
    n = 32
    rng = np.random.default_rng(seed)
    out = np.empty((hi - lo, n, n), dtype=np.float32)
    for s in range(0, hi, chunk):
        e = min(hi, s + chunk)
        blk = rng.standard_normal((e - s, n, n), dtype=np.float32)
        a, b = max(s, lo), e
        if b > a:
            out[a - lo:b - lo] = blk[a - s:b - s]
    return out


def gen_c3(batch: int = 262144, seed: int = 2, singular_frac: float = 0.01,
           chunk: int = C3_CHUNK, return_singular: bool = False):
    """BASELINE.json configs[2] under reading G15: A = (L·diag(u))[perm] with L unit-lower,
    strictly-lower N(0, std 0.5), u ~ U[0.5, 2]; then ⌊singular_frac·batch⌋ items get row j
    overwritten by row i (i ≠ j), making them exactly singular."""
    n = 64
    rng = np.random.default_rng(seed)
    A = np.empty((batch, n, n), dtype=np.float64)
    eye = np.eye(n)
    for s in range(0, batch, chunk):
        e = min(batch, s + chunk)
        m = e - s
        Ln = rng.normal(0.0, 0.5, (m, n, n))
        L = np.tril(Ln, -1) + eye
        u = rng.uniform(0.5, 2.0, (m, n))
        perm = rng.permuted(np.tile(np.arange(n), (m, 1)), axis=1)
        LU = L * u[:, None, :]
        A[s:e] = np.take_along_axis(LU, perm[:, :, None], axis=1)
    ns = int(np.floor(singular_frac * batch))
    S = np.sort(rng.choice(batch, ns, replace=False)) if ns > 0 else np.zeros(0, np.int64)
    for b in S:
        i, j = rng.choice(n, 2, replace=False)
        A[b, j] = A[b, i]
    return (A, S) if return_singular else A


def gen_gaussian(n: int, seed: int, dtype=np.float64) -> np.ndarray:
    """BASELINE.json configs[3]/[4] recipe: N(0,1)/sqrt(n) (C4: n=8192 seed 3; C5: n=32768 seed 4)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    A /= np.sqrt(n)
    return A.astype(dtype, copy=False)


def gen_c4(n: int = 8192, seed: int = 3) -> np.ndarray:
    return gen_gaussian(n, seed)


def gen_c5(n: int = 32768, seed: int = 4) -> np.ndarray:
    return gen_gaussian(n, seed)


def gen_normal_batch(batch: int, n: int, seed: int, dtype=np.float64) -> np.ndarray:
    """Generic i.i.d. N(0,1) batch (C2's recipe at other n / dtypes, for ragged-size tests)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, n, n)).astype(dtype)


# ---------------------------------------------------------------- exact companions

def sylvester_hadamard(n: int) -> np.ndarray:
    """H_1 = [1], H_2m = [[H, H], [H, -H]] (n a power of two)."""
    assert n >= 1 and (n & (n - 1)) == 0
    H = np.ones((1, 1))
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def hadamard_pd(n: int, seed: int = 5):
    """A = P·H·D (rows permuted by a seeded permutation, columns sign-flipped).
    Returns (A, perm, signs) with A[i] = H[perm[i]] * signs.  Exact inverse: D·Hᵀ·Pᵀ / n."""
    rng = np.random.default_rng(seed)
    H = sylvester_hadamard(n)
    perm = rng.permutation(n)
    signs = rng.choice(np.array([-1.0, 1.0]), n)
    A = H[perm] * signs[None, :]
    return np.ascontiguousarray(A), perm, signs


def permutation_matrix(perm) -> np.ndarray:
    """P with P[i, perm[i]] = 1."""
    n = len(perm)
    P = np.zeros((n, n))
    P[np.arange(n), np.asarray(perm)] = 1.0
    return P


def all_permutations(n: int) -> Iterator[tuple]:
    return itertools.permutations(range(n))


def signed_perm_pow2(n: int, seed: int = 7):
    """A = P·diag(±2^e), e ∈ [-8, 8] (P7): every GJ intermediate is exact in binary."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    e = rng.integers(-8, 9, n)
    s = rng.choice(np.array([-1.0, 1.0]), n)
    d = s * np.ldexp(1.0, e)
    A = np.zeros((n, n))
    A[np.arange(n), perm] = d[perm]
    return A, perm, d


def second_difference(n: int) -> np.ndarray:
    """tridiag(−1, 2, −1) (P8)."""
    return 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)


def hilbert(n: int) -> np.ndarray:
    """H_ij = 1/(i+j−1), 1-based."""
    i = np.arange(1, n + 1)
    return 1.0 / (i[:, None] + i[None, :] - 1)


def random_integer(n: int, seed: int, magnitude: int = 5) -> np.ndarray:
    """Integer entries in [−magnitude, magnitude], PCG64 seeded."""
    rng = np.random.default_rng(seed)
    return rng.integers(-magnitude, magnitude + 1, (n, n)).astype(np.float64)

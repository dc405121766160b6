"""Pins of the FULL-pivoting oracle (``oracle.invert_full_batched``, gj_oracle.c F1–F3;
PAPER.md Obs. 2–3, L59–L60) against things other than itself:

* LAPACK ``dgetc2`` (LU with complete pivoting) as a checker: the same row/column swap
  sequences and the same pivots (diag U) on random matrices — an independent library
  implementation of the same search;
* exact rational brute force (adjugate inverse, Laplace determinant);
* closed forms: permutation matrices (inverse = transpose, det = sign σ), Sylvester–
  Hadamard (exact inverse Aᵀ/n with ties at every step);
* hand-worked tie cases for reading G23 (first maximum in the row-major scan);
* the special case where complete and partial pivoting coincide (no swaps) against the
  pinned partial-pivoting oracle; singular flags.
"""
import math

import numpy as np
import pytest
import scipy.linalg.lapack as lapack

import oracle
import synth
from oracle import exact


def test_matches_lapack_getc2():
    rng = np.random.default_rng(21)
    for t in range(300):
        n = int(rng.integers(1, 25))
        A = rng.standard_normal((n, n))
        r = oracle.invert_full_batched(A)
        lu, ip, jp, info = lapack.dgetc2(A)
        assert info == 0
        assert np.array_equal(r.ipiv[0], ip + 1), t
        assert np.array_equal(r.jpiv[0], jp + 1), t
        np.testing.assert_allclose(r.pivots[0], np.diag(lu), rtol=1e-12, atol=0)
        s, ld = np.linalg.slogdet(A)
        assert r.sign[0] == s
        assert abs(r.logabsdet[0] - ld) <= 1e-11
        np.testing.assert_allclose(r.inverse[0], np.linalg.inv(A), rtol=0,
                                   atol=1e-12 * np.abs(np.linalg.inv(A)).max() * max(1.0, np.linalg.cond(A)))


def test_brute_force_rationals():
    rng = np.random.default_rng(22)
    checked = 0
    while checked < 200:
        n = int(rng.integers(1, 6))
        A = rng.integers(-4, 5, (n, n)).astype(float)
        d = exact.cofactor_det(A.tolist())
        r = oracle.invert_full_batched(A)
        if d == 0:
            assert r.info[0] != 0 or abs(r.det[0]) < 1e-12
            continue
        inv = np.array([[float(x) for x in row] for row in exact.adjugate_inverse(A.tolist())])
        kappa = np.abs(A).sum(1).max() * np.abs(inv).sum(1).max()
        assert r.info[0] == 0
        assert np.abs(r.inverse[0] - inv).max() <= kappa * 1e-16 * np.abs(inv).max() + 1e-18
        assert abs(r.det[0] - float(d)) <= 1e-15 * abs(float(d)) * kappa
        assert r.sign[0] == (1 if d > 0 else -1)
        checked += 1


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_all_permutation_matrices(n):
    for perm in synth.all_permutations(n):
        P = synth.permutation_matrix(perm)
        r = oracle.invert_full_batched(P)
        assert r.info[0] == 0
        assert np.array_equal(r.inverse[0], P.T)
        s = exact.permutation_sign(perm)
        assert r.det[0] == s and r.sign[0] == s and r.logabsdet[0] == 0.0


@pytest.mark.parametrize("n", [2, 8, 32])
def test_hadamard_exact(n):
    A, _, _ = synth.hadamard_pd(n, seed=5)
    r = oracle.invert_full_batched(A)
    assert r.info[0] == 0
    assert np.array_equal(r.inverse[0], A.T / n)
    assert abs(r.logabsdet[0] - 0.5 * n * math.log(n)) <= 1e-12 * n
    assert r.sign[0] == np.linalg.slogdet(A)[0]


def test_tie_rule_row_major_first():
    """G23 by hand: [[1, 2], [2, 1]]: |2| at (1, 2) and (2, 1) -> the row-major first,
    (1, 2): no row swap, columns 1 <-> 2; then the pivot 1 - 2*2/... = -3/2 at (2, 2)."""
    A = np.array([[1.0, 2.0], [2.0, 1.0]])
    r = oracle.invert_full_batched(A)
    assert r.ipiv[0].tolist() == [1, 2]
    assert r.jpiv[0].tolist() == [2, 2]
    assert r.pivots[0].tolist() == [2.0, 1.5]
    assert r.det[0] == -3.0 and r.sign[0] == -1
    # equal maxima in one row: the smallest column position wins
    B = np.array([[0.0, -3.0, 3.0], [1.0, 0.0, 0.0], [0.0, 1.0, 1.0]])
    rb = oracle.invert_full_batched(B)
    assert rb.ipiv[0, 0] == 1 and rb.jpiv[0, 0] == 2
    assert abs(rb.det[0] - np.linalg.det(B)) <= 1e-14


def test_no_swaps_equals_partial():
    """A matrix whose largest remaining entry is always the next diagonal one: complete and
    partial pivoting take the same steps, so the results agree with the pinned partial
    oracle bit for bit."""
    rng = np.random.default_rng(23)
    n = 12
    A = np.diag(2.0 ** -np.arange(n) * 64) + rng.uniform(-1e-3, 1e-3, (n, n))
    full = oracle.invert_full_batched(A)
    part = oracle.invert_batched(A)
    assert full.ipiv[0].tolist() == list(range(1, n + 1))
    assert full.jpiv[0].tolist() == list(range(1, n + 1))
    assert np.array_equal(full.inverse, part.inverse)
    assert np.array_equal(full.pivots, part.pivots)
    assert full.logabsdet[0] == part.logabsdet[0] and full.sign[0] == part.sign[0]


def test_singular_flags():
    r = oracle.invert_full_batched(np.array([[1.0, 2.0], [2.0, 4.0]]), tol=1e-12)
    assert r.info[0] == 2 and r.sign[0] == 0 and r.logabsdet[0] == -np.inf
    Z = np.zeros((3, 3))
    assert oracle.invert_full_batched(Z).info[0] == 1
    # rank 2 of 4: complete pivoting exhausts the rank, then step 3 fails
    rng = np.random.default_rng(24)
    U, V = rng.standard_normal((4, 2)), rng.standard_normal((2, 4))
    assert oracle.invert_full_batched(U @ V, tol=1e-12).info[0] == 3


def test_zero_pivot_recovered_by_column_swap():
    """Obs. 2: a zero in the pivot position is not singularity — here only a column
    swap (not a row swap) can bring a nonzero to it."""
    A = np.array([[0.0, 5.0], [0.0, 1.0]])
    assert oracle.invert_full_batched(A, tol=1e-12).info[0] == 2   # truly singular
    B = np.array([[0.0, 5.0], [1.0, 1.0]])
    r = oracle.invert_full_batched(B)
    assert r.ipiv[0, 0] == 1 and r.jpiv[0, 0] == 2
    assert np.allclose(r.inverse[0] @ B, np.eye(2), atol=1e-15)

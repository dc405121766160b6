"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against things other
than itself — the paper's worked matrix, exact rational brute force, closed forms, a
library special case (LAPACK getrf), mpmath at 50 digits and invariants.  Each test is
chosen so that a plausible mistake (dropped term, wrong sign, wrong index, transposed
operand, missing swap sign, wrong tie-break) fails at least one of them."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth
from oracle import exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _paper():
    with open(os.path.join(GOLD, "paper_3x3.json")) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- P1
def test_paper_matrix_exact():
    """P1: PAPER.md L89–L92 default matrix; values per BASELINE.json north_star."""
    g = _paper()
    r = oracle.invert_batched(np.array(g["A"], float))
    assert r.info[0] == 0
    assert np.array_equal(r.inverse[0], np.array(g["inverse"], float))  # bit-exact (dyadic)
    assert r.det[0] == g["det"]
    assert r.sign[0] == g["sign"]
    assert r.logabsdet[0] == g["logabsdet"]
    assert list(r.ipiv[0]) == g["ipiv"]
    assert list(r.pivots[0]) == g["pivots"]
    # reading G4: the unsigned Eq. (13) product is -1 on this matrix; det is +1
    assert np.prod(r.pivots[0]) == -1.0


def test_paper_matrix_brute_force_agrees_with_golden():
    """The golden values themselves, re-derived by the exact brute force (adjugate)."""
    g = _paper()
    inv = exact.adjugate_inverse(g["A"])
    assert [[int(x) for x in row] for row in inv] == g["inverse"]
    assert exact.cofactor_det(g["A"]) == g["det"]


def test_paper_step_one():
    """Eqs. (3)–(10)/(14)–(15) after step 1 on the paper matrix."""
    g = _paper()
    M = oracle.steps(np.array(g["A"], float), 1)
    assert np.array_equal(M, np.array(g["after_step_1_augmented"], float))
    # the listing's compact array = A^1 with its eliminated column replaced by D^1's column 1
    X = M[:, :3].copy()
    X[:, 0] = M[:, 3]
    assert np.array_equal(X, np.array(g["after_step_1_compact"], float))


def test_paper_matrix_without_pivoting():
    """Eqs. (3)–(10) literally (pivot = a_kk): pivots 1, 1, 1, same inverse."""
    g = _paper()
    r = oracle.invert_batched(np.array(g["A"], float), strategy="none")
    assert list(r.pivots[0]) == g["pivots_without_pivoting"]
    assert np.array_equal(r.inverse[0], np.array(g["inverse"], float))
    assert r.det[0] == 1.0


def test_paper_gap_diagnostics():
    g = _paper()
    r = oracle.invert_batched(np.array(g["A"], float))
    assert r.gap[0, 0] == 0.0          # three-way tie |1| = |1| = |1|
    assert r.gap[0, 1] == 0.5          # candidates |1|, |2|  -> (2-1)/2
    assert math.isinf(r.gap[0, 2])     # single candidate
    assert r.cmax_rel[0, 1] == 2.0 / 6.0


# ----------------------------------------------------------------------------- P2
def _int_sweep(count=500):
    """seeded integer matrices n = 2..6, entries in [-5, 5], |det| >= 1."""
    out = []
    seed = 0
    while len(out) < count:
        n = 2 + seed % 5
        A = synth.random_integer(n, seed=1000 + seed, magnitude=5)
        seed += 1
        d = exact.cofactor_det(A.tolist())
        if abs(d) >= 1:
            out.append((A, d))
    return out


def test_brute_force_sweep():
    """P2: oracle vs Laplace det and adjugate inverse in exact rationals (500 matrices)."""
    worst_inv = 0.0
    for A, d in _int_sweep():
        r = oracle.invert_batched(A)
        assert r.info[0] == 0
        inv = np.array([[float(x) for x in row] for row in exact.adjugate_inverse(A.tolist())])
        kappa = np.abs(A).sum(1).max() * np.abs(inv).sum(1).max()
        e = np.abs(r.inverse[0] - inv).max() / np.abs(inv).max()
        worst_inv = max(worst_inv, e / kappa)
        assert e <= kappa * 1e-16 + 1e-18, (A, e, kappa)
        assert abs(r.det[0] - float(d)) <= 1e-15 * max(1.0, abs(float(d))) * kappa
        assert r.sign[0] == (1 if d > 0 else -1)
        assert abs(r.logabsdet[0] - math.log(abs(d))) <= 1e-14 * kappa
    assert worst_inv < 1e-16


def test_brute_force_exhaustive_3x3_small():
    """SPEC.md L240ish 'oracle agreement': sampled 3×3 integer matrices in {-2..2}."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        A = rng.integers(-2, 3, (3, 3)).astype(float)
        d = exact.cofactor_det(A.tolist())
        r = oracle.invert_batched(A)
        if d == 0:
            assert r.info[0] != 0
            continue
        inv = np.array([[float(x) for x in row] for row in exact.adjugate_inverse(A.tolist())])
        assert np.abs(r.inverse[0] - inv).max() <= 1e-15 * np.abs(inv).max() * 50
        assert r.det[0] == float(d)


# ----------------------------------------------------------------------------- P3
def test_lapack_getrf_special_case():
    """P3: GJ partial-pivot ipiv == LAPACK getrf ipiv; pivots == diag(U); slogdet."""
    rng = np.random.default_rng(3)
    for t in range(200):
        n = int(rng.integers(1, 41))
        A = rng.standard_normal((n, n))
        r = oracle.invert_batched(A)
        lu, piv = scipy.linalg.lu_factor(A)
        # compare only up to the first near-tie (rule R3)
        for k in range(n):
            assert r.ipiv[0, k] == piv[k] + 1 or r.gap[0, k] <= 1e-6, (t, k)
            if r.ipiv[0, k] != piv[k] + 1:
                break
        else:
            np.testing.assert_allclose(r.pivots[0], np.diag(lu), rtol=1e-9, atol=0)
        s, ld = np.linalg.slogdet(A)
        assert r.sign[0] == s
        assert abs(r.logabsdet[0] - ld) <= 1e-10


# ----------------------------------------------------------------------------- P5
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_all_permutation_matrices(n):
    """P5: inverse = transpose exactly, det = sign(σ) exactly."""
    for perm in synth.all_permutations(n):
        P = synth.permutation_matrix(perm)
        r = oracle.invert_batched(P)
        assert r.info[0] == 0
        assert np.array_equal(r.inverse[0], P.T)
        s = exact.permutation_sign(perm)
        assert r.det[0] == s and r.sign[0] == s and r.logabsdet[0] == 0.0


# ----------------------------------------------------------------------------- P6
@pytest.mark.parametrize("n", [2, 16, 64, 256])
def test_hadamard_exact(n):
    """P6: A = P·H·D; exact inverse D·Hᵀ·Pᵀ/n, logabsdet = (n/2)·ln n, every step a tie."""
    A, perm, signs = synth.hadamard_pd(n, seed=5)
    r = oracle.invert_batched(A)
    assert r.info[0] == 0
    expect = (A.T / n)  # (PHD)^-1 = D H^T P^T / n = A^T / n since H^T H = n I
    assert np.array_equal(r.inverse[0], expect)
    assert abs(r.logabsdet[0] - 0.5 * n * math.log(n)) <= 1e-12 * n
    pv = np.abs(r.pivots[0])
    assert np.all(np.log2(pv) == np.round(np.log2(pv)))  # powers of two
    lu, piv = scipy.linalg.lu_factor(A)
    assert np.array_equal(r.ipiv[0], piv + 1)
    s, _ = np.linalg.slogdet(A)
    assert r.sign[0] == s


# ----------------------------------------------------------------------------- P7
def test_signed_permutation_pow2():
    A, perm, d = synth.signed_perm_pow2(64, seed=7)
    r = oracle.invert_batched(A)
    expect = np.zeros_like(A)
    expect[perm, np.arange(64)] = 1.0 / d[perm]
    assert np.array_equal(r.inverse[0], expect)


# ----------------------------------------------------------------------------- P8
@pytest.mark.parametrize("n", [1, 5, 50])
def test_second_difference_closed_form(n):
    """P8: det tridiag(-1,2,-1) = n+1; A^-1_ij = min(i,j)(n+1-max(i,j))/(n+1); no swaps."""
    A = synth.second_difference(n)
    r = oracle.invert_batched(A)
    i = np.arange(1, n + 1)
    expect = np.minimum.outer(i, i) * (n + 1 - np.maximum.outer(i, i)) / (n + 1)
    assert np.abs(r.inverse[0] - expect).max() <= 1e-15 * n * n
    assert abs(r.det[0] - (n + 1)) <= 1e-14 * n
    assert np.array_equal(r.ipiv[0], i)
    np.testing.assert_allclose(r.pivots[0], (i + 1) / i, rtol=1e-16)


# ----------------------------------------------------------------------------- P9
def _hilbert_inverse(n):
    from math import comb
    H = np.empty((n, n))
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            H[i - 1, j - 1] = ((-1) ** (i + j) * (i + j - 1) * comb(n + i - 1, n - j)
                               * comb(n + j - 1, n - i) * comb(i + j - 2, i - 1) ** 2)
    return H


@pytest.mark.parametrize("n", [1, 2, 4, 6, 8])
def test_hilbert_closed_form(n):
    """P9: textbook integer inverse of the Hilbert matrix."""
    A = synth.hilbert(n)
    r = oracle.invert_batched(A)
    expect = _hilbert_inverse(n)
    kappa = oracle.kappa_inf(A, expect)[0]
    e = np.abs(r.inverse[0] - expect).max() / np.abs(expect).max()
    # input rounding of 1/(i+j-1) to fp64 perturbs A by ~1e-16 relative => error <= kappa*eps64
    assert e <= kappa * 2.3e-16


# ----------------------------------------------------------------------------- P10
def test_mpmath_50_digits():
    """P10: long-double oracle vs mpmath at 50 digits, n <= 12: agreement <= kappa*1e-18."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    rng = np.random.default_rng(10)
    for n in (2, 5, 9, 12):
        for _ in range(3):
            A = rng.standard_normal((n, n))
            r = oracle.invert_batched(A)
            M = mp.matrix(A.tolist())
            Minv = M ** -1
            inv = np.array([[float(Minv[i, j]) for j in range(n)] for i in range(n)])
            kappa = oracle.kappa_inf(A, inv)[0]
            e = np.abs(r.inverse[0] - inv).max() / np.abs(inv).max()
            assert e <= kappa * 1e-18 + 2.3e-16   # + the final rounding to fp64
            d = float(mp.det(M))
            assert abs(r.det[0] - d) <= abs(d) * (kappa * 1e-18 + 2.3e-16)


# ----------------------------------------------------------------------------- singular / Obs. 2
def test_singular_rank_one():
    """[[1,2],[2,4]] is singular; step 2 fails."""
    r = oracle.invert_batched(np.array([[1.0, 2.0], [2.0, 4.0]]), tol=1e-12)
    assert r.info[0] == 2 and r.sign[0] == 0 and r.det[0] == 0.0 and r.logabsdet[0] == -np.inf


def test_zero_pivot_is_not_singular():
    """Obs. 2: a zero pivot does not imply singularity."""
    A = np.array([[0.0, 1.0], [1.0, 0.0]])
    none = oracle.invert_batched(A, strategy="none")
    assert none.info[0] == 1
    part = oracle.invert_batched(A)
    assert part.info[0] == 0
    assert np.array_equal(part.inverse[0], A) and part.det[0] == -1.0 and part.sign[0] == -1


def test_zero_column_exact_threshold():
    r = oracle.invert_batched(np.array([[0.0, 1.0], [0.0, 1.0]]), tol=0.0)
    assert r.info[0] == 1


def test_duplicated_row_flagged_relative_threshold():
    """Reading G1: duplicated-row items are flagged at tol = 1e-10 relative (C3's recipe)."""
    A, S = synth.gen_c3(batch=400, return_singular=True)
    r = oracle.invert_batched(A, tol=synth.C3_TOL)
    flagged = np.nonzero(r.info)[0]
    assert np.array_equal(flagged, S)
    assert np.all(r.sign[S] == 0)


# ----------------------------------------------------------------------------- tie-break (G3)
def test_tie_break_smallest_row():
    A = np.array([[0.0, 0.0, 1.0], [2.0, 1.0, 0.0], [-2.0, 0.0, 1.0]])
    r = oracle.invert_batched(A)
    assert r.ipiv[0, 0] == 2       # |2| = |-2| tie -> row 2 (1-based), not 3
    A2 = np.array([[1.0, 0.0], [-1.0, 1.0]])
    assert oracle.invert_batched(A2).ipiv[0, 0] == 1


# ----------------------------------------------------------------------------- P4 invariants
def test_invariants():
    rng = np.random.default_rng(4)
    for n in (3, 7, 16, 33):
        A = rng.standard_normal((n, n))
        r = oracle.invert_batched(A)
        X = r.inverse[0]
        assert oracle.residual(A, X) <= 1e-12
        assert np.abs(X @ A - np.eye(n)).max() <= 1e-12
        # det(PA) = sign(P) det A
        perm = rng.permutation(n)
        rp = oracle.invert_batched(A[perm])
        assert abs(rp.logabsdet[0] - r.logabsdet[0]) <= 1e-13
        assert rp.sign[0] == r.sign[0] * exact.permutation_sign(perm)
        # inverse of PA = A^-1 P^T
        assert np.abs(rp.inverse[0] - X[:, perm]).max() <= 1e-12 * np.abs(X).max()
        # det(A^T) = det(A)
        rt = oracle.invert_batched(A.T.copy())
        assert abs(rt.logabsdet[0] - r.logabsdet[0]) <= 1e-13 and rt.sign[0] == r.sign[0]
        # logdet(cA) = logdet(A) + n log|c|
        rc = oracle.invert_batched(-2.5 * A)
        assert abs(rc.logabsdet[0] - (r.logabsdet[0] + n * math.log(2.5))) <= 1e-12
        assert rc.sign[0] == r.sign[0] * (-1) ** n
        # involution
        rr = oracle.invert_batched(X)
        assert np.abs(rr.inverse[0] - A).max() <= 1e-10


def test_batch_order_invariance():
    A = synth.gen_normal_batch(64, 9, seed=12)
    r = oracle.invert_batched(A)
    perm = np.random.default_rng(1).permutation(64)
    rp = oracle.invert_batched(A[perm])
    assert np.array_equal(rp.inverse, r.inverse[perm]) and np.array_equal(rp.ipiv, r.ipiv[perm])


def test_single_matrix_threads_equal_batched():
    A = synth.gen_gaussian(96, seed=3)
    r1 = oracle.invert(A, nthreads=4)
    r2 = oracle.invert_batched(A)
    assert np.array_equal(r1.inverse, r2.inverse) and np.array_equal(r1.ipiv, r2.ipiv)


def test_rejects_non_finite():
    with pytest.raises(ValueError):
        oracle.invert_batched(np.array([[np.nan]]))


def test_fp32_inputs_widen_exactly():
    A = synth.gen_normal_batch(8, 5, seed=2, dtype=np.float32)
    r32 = oracle.invert_batched(A)
    r64 = oracle.invert_batched(A.astype(np.float64))
    assert np.array_equal(r32.inverse, r64.inverse)


def test_c1_item0_is_paper_block():
    A = synth.gen_c1(batch=8)
    r = oracle.invert_batched(A)
    exp = np.eye(16)
    exp[:3, :3] = _paper()["inverse"]
    assert np.array_equal(r.inverse[0], exp)
    assert list(r.ipiv[0]) == [1, 3, 3] + list(range(4, 17))
    assert r.det[0] == 1.0

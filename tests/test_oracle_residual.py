"""Pins for the oracle's residual functions (``gjo_residual_rows`` / ``gjo_residual_batched``),
which judge rule R2 (max |A·X − I|, reading G17; the property is Eq. (12), A⁻¹ = Dⁿ,
PAPER.md L52) on C1–C5.

The expected values never come from the oracle: A is a product of integer elementary
matrices, so its inverse X0 is the reverse product of the inverted factors, exact in
integers; X = X0 + E with dyadic entries in E, so A·X − I = A·E holds exactly and its
maximum is computed here in Python integers/Fractions.  E is placed so that each row has a
different residual, which makes a dropped row, a wrong row index, a transposed product, a
missing −δ_ij or a reduction that keeps the wrong maximum visible."""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def _unimodular(n, rng, nfac=None):
    """(A, A^-1) as exact int64 matrices: A = F_1 ... F_m with F = I + c e_i e_j^T (i != j)."""
    A = np.eye(n, dtype=np.int64)
    X = np.eye(n, dtype=np.int64)
    for _ in range(nfac or (3 * n if n > 1 else 0)):
        i, j = rng.choice(n, 2, replace=False)
        c = int(rng.integers(-2, 3)) or 1
        F = np.eye(n, dtype=np.int64)
        F[i, j] = c
        Fi = np.eye(n, dtype=np.int64)
        Fi[i, j] = -c
        A = A @ F
        X = Fi @ X
        if np.abs(A).max() > 2 ** 20 or np.abs(X).max() > 2 ** 20:   # stay far inside doubles
            A = A @ Fi
            X = F @ X
    assert np.array_equal(A @ X, np.eye(n, dtype=np.int64))
    return A, X


def _exact_residual(A, X, rows=None):
    """max_{i in rows, j} |(A X)_ij - delta_ij| in exact rationals."""
    n = A.shape[0]
    Af = [[Fraction(int(v)) for v in row] for row in A]
    Xf = [[Fraction(float(v)) for v in row] for row in X]
    worst = Fraction(0)
    for i in (range(n) if rows is None else rows):
        for j in range(n):
            s = sum(Af[i][k] * Xf[k][j] for k in range(n)) - (1 if i == j else 0)
            worst = max(worst, abs(s))
    return worst


def test_exact_inverse_has_zero_residual():
    rng = np.random.default_rng(11)
    for n in (1, 2, 5, 16, 33):
        A, X = _unimodular(n, rng)
        assert oracle.residual(A.astype(float), X.astype(float)) == 0.0


def test_identity_terms_are_subtracted_on_the_diagonal_only():
    """X = 0 gives max |-I| = 1; X = 2 A^-1 gives A X - I = I (max 1); X = A^-1 gives 0."""
    rng = np.random.default_rng(12)
    A, X = _unimodular(7, rng)
    Ad = A.astype(float)
    assert oracle.residual(Ad, np.zeros((7, 7))) == 1.0
    assert oracle.residual(Ad, 2.0 * X.astype(float)) == 1.0
    assert oracle.residual(np.eye(7), 3.0 * np.eye(7)) == 2.0


@pytest.mark.parametrize("n", [3, 8, 20])
def test_perturbed_inverse_exact_value(n):
    """One dyadic perturbation per column of X: (A E)_ij = A[i, p_j] e_j, known exactly."""
    rng = np.random.default_rng(100 + n)
    A, X0 = _unimodular(n, rng)
    E = np.zeros((n, n))
    for j in range(n):
        E[rng.integers(n), j] = float(rng.integers(1, 8)) * 2.0 ** -int(rng.integers(10, 30))
    X = X0.astype(float) + E
    assert np.array_equal(X - X0, E)   # X is exact in doubles
    got = oracle.residual(A.astype(float), X)
    assert Fraction(got) == _exact_residual(A, X)
    assert got > 0.0


def test_rows_subset_and_row_identity():
    """Each row gets a distinct residual; the rows argument must select exactly those rows."""
    rng = np.random.default_rng(7)
    n = 9
    A = np.eye(n, dtype=np.int64)            # A = I: (A E) = E, row i's residual = max |E_i.|
    X0 = np.eye(n, dtype=np.int64)
    E = np.zeros((n, n))
    for i in range(n):
        E[i, rng.integers(n)] = 2.0 ** -(i + 3)   # row i: 2^-(i+3), all distinct
    X = X0 + E
    for rows in ([0], [8], [3, 5], [8, 2, 6], list(range(n))):
        want = max(2.0 ** -(i + 3) for i in rows)
        assert oracle.residual(A.astype(float), X, rows=rows) == want
    # a general unimodular A: subsets against the exact rationals
    A, X0 = _unimodular(n, rng)
    X = X0.astype(float) + E
    for rows in ([1], [4, 7], [0, 8]):
        assert Fraction(oracle.residual(A.astype(float), X, rows=rows)) == _exact_residual(A, X, rows)


def test_operand_order_matters():
    """max|A E| = 1/16 but max|E A| = 3/16 here: computing X·A instead of A·X would fail."""
    A = np.array([[1, 3], [0, 1]], dtype=np.int64)
    X0 = np.array([[1, -3], [0, 1]], dtype=np.int64)
    E = np.array([[2.0 ** -4, 0.0], [0.0, 0.0]])
    X = X0 + E
    assert _exact_residual(A, X) == Fraction(1, 16)
    assert oracle.residual(A.astype(float), X) == 2.0 ** -4
    assert oracle.residual(X, A.astype(float)) == 3 * 2.0 ** -4   # X A - I = E A


def test_batched_matches_per_item_exact_values():
    rng = np.random.default_rng(5)
    n, B = 6, 40
    As, Xs, want = [], [], []
    for b in range(B):
        A, X0 = _unimodular(n, rng)
        E = np.zeros((n, n))
        E[b % n, (3 * b) % n] = 2.0 ** -(b % 20 + 5)
        X = X0.astype(float) + E
        As.append(A.astype(float))
        Xs.append(X)
        want.append(_exact_residual(A, X))
    out = oracle.residual_batched(np.array(As), np.array(Xs))
    assert [Fraction(v) for v in out] == want
    # item order: the b-th output belongs to the b-th item
    out_rev = oracle.residual_batched(np.array(As[::-1]), np.array(Xs[::-1]))
    assert np.array_equal(out_rev, out[::-1])

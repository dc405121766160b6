"""Pins of the multi-RHS oracle (``oracle.solve_batched``, gjo_solve: Gauss–Jordan on
[A | B]) against things other than itself: B = I reproduces the pinned
inverse oracle bit for bit (the same operations on the same columns), exact rationals
(adjugate · B), LAPACK gesv / getrf as checkers, and the residual."""
import numpy as np
import scipy.linalg

import oracle
from oracle import exact


def test_identity_rhs_is_the_inverse():
    rng = np.random.default_rng(60)
    for n in (1, 2, 5, 16, 33):
        A = rng.standard_normal((20, n, n))
        s = oracle.solve_batched(A, np.broadcast_to(np.eye(n), (20, n, n)))
        r = oracle.invert_batched(A)
        assert np.array_equal(s.X, r.inverse)
        assert np.array_equal(s.ipiv, r.ipiv)
        assert np.array_equal(s.logabsdet, r.logabsdet) and np.array_equal(s.sign, r.sign)


def test_exact_rationals():
    rng = np.random.default_rng(61)
    done = 0
    while done < 150:
        n = int(rng.integers(1, 6))
        m = int(rng.integers(1, 4))
        A = rng.integers(-4, 5, (n, n)).astype(float)
        B = rng.integers(-4, 5, (n, m)).astype(float)
        d = exact.cofactor_det(A.tolist())
        if d == 0:
            continue
        inv = exact.adjugate_inverse(A.tolist())
        Xe = np.array([[float(sum(inv[i][k] * int(B[k, j]) for k in range(n))) for j in range(m)] for i in range(n)])
        s = oracle.solve_batched(A, B)
        assert s.info[0] == 0
        kappa = np.abs(A).sum(1).max() * np.abs(np.array([[float(x) for x in r] for r in inv])).sum(1).max()
        assert np.abs(s.X[0] - Xe).max() <= kappa * 1e-16 * max(1.0, np.abs(Xe).max())
        done += 1


def test_lapack_checkers():
    rng = np.random.default_rng(62)
    for t in range(100):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(1, 9))
        A = rng.standard_normal((n, n))
        B = rng.standard_normal((n, m))
        s = oracle.solve_batched(A, B)
        X = scipy.linalg.solve(A, B)
        kappa = np.linalg.cond(A, np.inf)
        assert np.abs(s.X[0] - X).max() <= 1e-14 * kappa * max(1.0, np.abs(X).max())
        _, piv = scipy.linalg.lu_factor(A)
        for k in range(n):
            if s.ipiv[0, k] != piv[k] + 1:
                assert s.gap[0, k] <= 1e-6
                break
        sg, ld = np.linalg.slogdet(A)
        assert s.sign[0] == sg and abs(s.logabsdet[0] - ld) <= 1e-10
        assert oracle.residual(A, np.linalg.inv(A)) < 1e-10


def test_singular_flag():
    A = np.array([[1.0, 2.0], [2.0, 4.0]])
    s = oracle.solve_batched(A, np.ones((2, 3)), tol=1e-12)
    assert s.info[0] == 2 and s.sign[0] == 0 and np.all(np.isnan(s.X[0]))

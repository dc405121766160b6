"""Pivoting strategies on the GPU (gj_invert_batched_pivoting, K6):
parity of "none" (Eqs. (3)–(10), pivot a_kk) and "partial" (the listing) against the
oracle's strategies, and the paper's §4 claim — pivoting reduces rounding error (Obs. 3,
PAPER.md L60; L207) — on matrix families where the ordering is known from the theory:

* tiny leading pivots: no pivoting divides by them; partial pivoting does not;
* Wilkinson's growth matrix (1 on the diagonal and in the last column, -1 below the
  diagonal): partial pivoting takes no row swaps and the last column grows as 2^(n-1);
  full pivoting keeps the growth small.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.parity import assert_report, compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def gj():
    import paper_1401_7962_b200 as g
    return g


def run(gj, torch, A, strategy, tol=None):
    r = gj.invert_batched_pivoting(torch.from_numpy(np.ascontiguousarray(A)).cuda(), strategy, tol)
    torch.cuda.synchronize()
    return {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}


def eps(dtype):
    return 2.0 ** -23 if dtype == np.float32 else 2.0 ** -52


@pytest.mark.parametrize("n", [1, 3, 8, 17, 32])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_none_vs_oracle(gj, torch, n, dtype):
    """Diagonally dominant inputs, where pivot a_kk is safe: "none" against the oracle's
    strategy 0 (ipiv = 1..n, jpiv = 1..n)."""
    rng = np.random.default_rng(400 + n)
    B = 777
    A = (rng.uniform(-1, 1, (B, n, n)) + 2 * n * np.eye(n)).astype(dtype)
    tol = n * eps(dtype)
    g = run(gj, torch, A, "none", tol)
    ref = oracle.invert_batched(A, tol=tol, strategy="none")
    assert np.all(g["ipiv"] == np.arange(1, n + 1)) and np.all(g["jpiv"] == np.arange(1, n + 1))
    rep = compare(A, g, ref, dtype, tol, flat_only=True)
    print(rep.summary())
    assert_report(rep, flat_only=True)


@pytest.mark.parametrize("n", [2, 7, 16, 29, 32])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_partial_vs_oracle(gj, torch, n, dtype):
    A = synth.gen_normal_batch(1037, n, seed=500 + n, dtype=dtype)
    tol = n * eps(dtype)
    g = run(gj, torch, A, "partial", tol)
    ref = oracle.invert_batched(A, tol=tol)
    assert np.all(g["jpiv"] == np.arange(1, n + 1))
    rep = compare(A, g, ref, dtype, tol)
    print(rep.summary())
    assert_report(rep)


def test_zero_pivot_obs2(gj, torch):
    """Obs. 2: a zero pivot does not mean singular — "none" fails at step 1, the pivoting
    strategies invert exactly."""
    A = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert run(gj, torch, A, "none")["info"] == 1
    for s in ("partial", "full"):
        g = run(gj, torch, A, s)
        assert g["info"] == 0 and np.array_equal(g["inverse"], A) and g["sign"] == -1


def _residual(A, X):
    return oracle.residual_batched(A.astype(np.float64), X.astype(np.float64))


def test_tiny_pivots_need_pivoting(gj, torch):
    rng = np.random.default_rng(41)
    B, n = 256, 16
    A = rng.standard_normal((B, n, n)).astype(np.float32)
    A[:, 0, 0] = 1e-6 * rng.standard_normal(B).astype(np.float32)   # tiny leading pivot
    res = {s: _residual(A, run(gj, torch, A, s)["inverse"]) for s in ("none", "partial", "full")}
    med = {s: float(np.median(v)) for s, v in res.items()}
    print("median residuals:", med)
    assert med["none"] > 100 * med["partial"]
    assert med["full"] <= 4 * med["partial"]


@pytest.mark.parametrize("n", [24, 32])
def test_wilkinson_growth_needs_full(gj, torch, n):
    rng = np.random.default_rng(42)
    W = np.broadcast_to(np.eye(n) - np.tril(np.ones((n, n)), -1), (64, n, n)).copy()
    # a random last column (inexact values: with all-ones the growth is in powers of two
    # and exact) and random signs D1 W D2 (the same magnitudes, so the same ties and the
    # same 2^(n-1) growth under partial pivoting)
    W[:, :, -1] = rng.uniform(0.5, 1.0, (64, n))
    d1 = rng.choice([-1.0, 1.0], (64, n, 1))
    d2 = rng.choice([-1.0, 1.0], (64, 1, n))
    A = (d1 * W * d2).astype(np.float32)
    X_ref = oracle.invert_full_batched(A).inverse
    err = {}
    for s in ("partial", "full"):
        X = run(gj, torch, A, s)["inverse"].astype(np.float64)
        err[s] = float(np.median(np.abs(X - X_ref).max(axis=(1, 2)) / np.abs(X_ref).max(axis=(1, 2))))
    print(f"n={n} median relative error: {err}")
    assert err["partial"] > 1000 * err["full"]

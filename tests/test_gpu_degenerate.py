"""Degenerate items through every batched entry point: an all-zero matrix (every pivot 0:
1/p is infinite and the item's rows turn into NaN after the first step), next to an
identity and a Gaussian item in the same warp task.  Nothing may fault, the zero item is
flagged at step 1 with sign 0 and log|det| = -inf, and its neighbours are exact / correct.
(Found by tools/fuzz_batched.py: the full-pivoting kernel's column search compared NaN keys
of different payloads and indexed out of range.)"""
import numpy as np
import pytest

import oracle

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


def batch(n, dtype):
    A = np.zeros((3, n, n), dtype)
    A[1] = np.eye(n)
    A[2] = np.random.default_rng(n).standard_normal((n, n))
    return A


def check(r, A, dtype):
    info = r.info.cpu().numpy()
    assert info[0] == 1 and info[1] == 0 and info[2] == 0
    assert r.sign.cpu().numpy()[0] == 0 and np.isneginf(r.logabsdet.cpu().numpy()[0])
    assert r.logabsdet.cpu().numpy()[1] == 0.0


@pytest.mark.parametrize("n", [1, 2, 5, 8, 16, 32, 33, 64])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_zero_item_every_entry(gj, torch, n, dtype):
    A = batch(n, dtype)
    At = torch.from_numpy(A).cuda()
    tol = float(n * (2.0 ** -23 if dtype == np.float32 else 2.0 ** -52))
    r = gj.invert_batched(At, tol=tol)
    d = gj.det(At, tol=tol)
    torch.cuda.synchronize()
    check(r, A, dtype)
    check(d, A, dtype)
    assert np.array_equal(r.inverse.cpu().numpy()[1], np.eye(n, dtype=dtype))
    ref = oracle.invert_batched(A[2:], tol=tol)
    e = np.abs(r.inverse.cpu().numpy()[2] - ref.inverse[0]).max() / np.abs(ref.inverse[0]).max()
    kap = np.abs(A[2]).sum(1).max() * np.abs(ref.inverse[0]).sum(1).max()
    assert e <= max(1e-10 if dtype == np.float64 else 2e-4, kap * tol / n)
    if n <= 32:
        for m in (1, 3, 8, 32):
            B = np.ones((3, n, m), dtype)
            s = gj.solve_batched(At, torch.from_numpy(B).cuda(), tol=tol)
            torch.cuda.synchronize()
            check(s, A, dtype)
            assert np.array_equal(s.X.cpu().numpy()[1], B[1])
        for strat in ("none", "partial", "full"):
            f = gj.invert_batched_pivoting(At, strategy=strat, tol=tol)
            torch.cuda.synchronize()
            check(f, A, dtype)
            assert np.array_equal(f.inverse.cpu().numpy()[1], np.eye(n, dtype=dtype))

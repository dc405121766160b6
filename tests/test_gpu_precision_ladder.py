"""the precision ladder: against the long-double oracle, every GPU path's
relative inverse error stays within a small constant of kappa_inf * eps of its dtype:
e <= 0.12 kappa eps for both dtypes (reading G25 of DESIGN.md: SURVEY's probe constant
0.015 for fp64 is exceeded by the maximum over 2,000 Gaussian items of every fp64 path,
~0.06 — the same ratio the fp32 paths show); a ratio far above it means a bug, not
rounding (the parity rule R1 allows 1.0).
Measured on Gaussian inputs through each kernel family (K1/K1b, K2/K2b, K6, K7, the
blocked large-n path in both dtypes)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

LADDER = {np.float64: (0.12, 2.0 ** -52), np.float32: (0.12, 2.0 ** -23)}


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def gj():
    import paper_1401_7962_b200 as g
    return g


def ratio(A, X, Xr, dtype):
    A = np.asarray(A, np.float64)
    Xr = np.asarray(Xr, np.float64)
    kappa = np.abs(A).sum(-1).max(-1) * np.abs(Xr).sum(-1).max(-1)
    e = np.abs(np.asarray(X, np.float64) - Xr).max(axis=(-2, -1)) / np.abs(Xr).max(axis=(-2, -1))
    return e / (kappa * LADDER[dtype][1])


def check(r, dtype, what):
    c = LADDER[dtype][0]
    print(f"{what}: max e/(kappa eps) = {np.max(r):.4f} (ladder {c})")
    assert np.max(r) <= c, what


@pytest.mark.parametrize("n,dtype", [(16, np.float64), (32, np.float32), (32, np.float64), (48, np.float32),
                                     (64, np.float64), (64, np.float32)])
def test_batched(gj, torch, n, dtype):
    A = synth.gen_normal_batch(2000, n, seed=1100 + n, dtype=dtype)
    r = gj.invert_batched(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    ref = oracle.invert_batched(A)
    ok = (ref.info == 0) & (r.info.cpu().numpy() == 0)
    check(ratio(A[ok], r.inverse.cpu().numpy()[ok], ref.inverse[ok], dtype), dtype, f"batched n={n} {dtype.__name__}")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_full_pivoting_and_solve(gj, torch, dtype):
    n = 32
    A = synth.gen_normal_batch(2000, n, seed=1200, dtype=dtype)
    At = torch.from_numpy(A).cuda()
    rf = gj.invert_batched_full(At)
    torch.cuda.synchronize()
    ref = oracle.invert_full_batched(A)
    check(ratio(A, rf.inverse.cpu().numpy(), ref.inverse, dtype), dtype, f"full pivoting {dtype.__name__}")
    B = np.broadcast_to(np.eye(n, dtype=dtype), (2000, n, n)).copy()
    rs = gj.solve_batched(At, torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    check(ratio(A, rs.X.cpu().numpy(), ref.inverse, dtype), dtype, f"solve B=I {dtype.__name__}")


@pytest.mark.parametrize("n,dtype", [(300, np.float64), (1024, np.float64), (300, np.float32), (1024, np.float32)])
def test_large(gj, torch, n, dtype):
    A = synth.gen_gaussian(n, seed=1300 + n).astype(dtype)
    r = gj.invert(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    ref = oracle.invert(A)
    check(ratio(A, r.inverse.cpu().numpy(), ref.inverse[0], dtype), dtype, f"large n={n} {dtype.__name__}")

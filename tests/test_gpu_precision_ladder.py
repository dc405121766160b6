"""the precision ladder: against the long-double oracle, every GPU path's
relative inverse error e = max|X - X_ref| / max|X_ref| stays within a small constant c of
kappa_inf * eps of its dtype (the parity rule R1 allows c = 1).

Reading G25: c is set PER PATH to 1.5x the maximum measured over the test's
seeded inputs (round 2, 1x B200; the inputs and the kernels are deterministic, so the
measured value is exact), so an error that doubles fails.  SURVEY's 0.015 for fp64 does not
describe this statistic: `tools/ladder_probe.c` runs the TEXTBOOK fp64 Gauss-Jordan (per-
element division, no FMA) on 2,000 Gaussian items and gets max e/(kappa eps) = 0.119
(n = 16), 0.079-0.086 (n = 32), 0.066 (n = 64) — the GPU fp64 paths (0.06-0.10) sit at the
textbook algorithm's own level, not above it.  The large-n paths (blocked, 128-column
panels) are much lower because kappa_inf of an n = 300..1024 Gaussian matrix grows faster
than the max-entry error.
Measured on Gaussian inputs through each kernel family (K1/K1b, K2/K2f, K6, K7/K1s, the
blocked large-n path in both dtypes)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

EPS = {np.float64: 2.0 ** -52, np.float32: 2.0 ** -23}
# measured max e/(kappa eps), round 2 (gpurun_out/ladder.log -> DESIGN.md G25); constant = 1.5x
MEASURED = {
    ("batched", 16, np.float64): 0.0993, ("batched", 32, np.float32): 0.0770,
    ("batched", 32, np.float64): 0.0647, ("batched", 48, np.float32): 0.0658,
    ("batched", 64, np.float64): 0.0618, ("batched", 64, np.float32): 0.0551,
    ("full", 32, np.float32): 0.0633, ("full", 32, np.float64): 0.0602,
    ("solve", 32, np.float32): 0.0814, ("solve", 32, np.float64): 0.0774,
    ("large", 300, np.float64): 0.0105, ("large", 1024, np.float64): 0.0169,
    ("large", 300, np.float32): 0.0061, ("large", 1024, np.float32): 0.0144,
}
MARGIN = 1.5


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
    return e / (kappa * EPS[dtype])


def check(r, key, what):
    c = MARGIN * MEASURED[key]
    print(f"{what}: max e/(kappa eps) = {np.max(r):.4f} (ladder {c:.4f})")
    assert np.max(r) <= c, what


@pytest.mark.parametrize("n,dtype", [(16, np.float64), (32, np.float32), (32, np.float64), (48, np.float32),
                                     (64, np.float64), (64, np.float32)])
def test_batched(gj, torch, n, dtype):
    A = synth.gen_normal_batch(2000, n, seed=1100 + n, dtype=dtype)
    r = gj.invert_batched(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    ref = oracle.invert_batched(A)
    ok = (ref.info == 0) & (r.info.cpu().numpy() == 0)
    check(ratio(A[ok], r.inverse.cpu().numpy()[ok], ref.inverse[ok], dtype), ("batched", n, dtype),
          f"batched n={n} {dtype.__name__}")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_full_pivoting_and_solve(gj, torch, dtype):
    n = 32
    A = synth.gen_normal_batch(2000, n, seed=1200, dtype=dtype)
    At = torch.from_numpy(A).cuda()
    rf = gj.invert_batched_full(At)
    torch.cuda.synchronize()
    ref = oracle.invert_full_batched(A)
    check(ratio(A, rf.inverse.cpu().numpy(), ref.inverse, dtype), ("full", n, dtype), f"full pivoting {dtype.__name__}")
    B = np.broadcast_to(np.eye(n, dtype=dtype), (2000, n, n)).copy()
    rs = gj.solve_batched(At, torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    check(ratio(A, rs.X.cpu().numpy(), ref.inverse, dtype), ("solve", n, dtype), f"solve B=I {dtype.__name__}")


@pytest.mark.parametrize("n,dtype", [(300, np.float64), (1024, np.float64), (300, np.float32), (1024, np.float32)])
def test_large(gj, torch, n, dtype):
    A = synth.gen_gaussian(n, seed=1300 + n).astype(dtype)
    r = gj.invert(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    ref = oracle.invert(A)
    check(ratio(A, r.inverse.cpu().numpy(), ref.inverse[0], dtype), ("large", n, dtype), f"large n={n} {dtype.__name__}")

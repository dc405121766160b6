"""K1s (gj_batched.cu): the blocked fp32 n = 32 elimination without the D half, used by
gj_solve_batched for 1 <= nrhs <= 8 and by the determinant-only run (gj_det / inverse=False).
  * solve: parity with the [A | B] oracle on the kappa-scaled rule (R1), ragged batches (a
    padding matrix in the last two-matrix task), singular items, exact pins;
  * det-only: log|det|, sign, det, ipiv and info bitwise equal to the inverting path (K1b) —
    the two share every pivot-chain operation, so the pivots are the same numbers;
  * K7 (more than 8 right-hand sides at n = 32) agrees with the oracle."""
import os
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EPS = 2.0 ** -23


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def gj():
    import paper_1401_7962_b200 as g
    return g


def solve(gj, torch, A, B, tol):
    r = gj.solve_batched(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), tol=tol)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in r._asdict().items()}


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("batch", [1, 2, 1001])
def test_solve_vs_oracle(gj, torch, m, batch):
    A = synth.gen_normal_batch(batch, 32, seed=40 + m, dtype=np.float32)
    B = np.random.default_rng(50 + m).standard_normal((batch, 32, m)).astype(np.float32)
    tol = 32 * EPS
    g = solve(gj, torch, A, B, tol)
    ref = oracle.solve_batched(A, B, tol=tol)
    ok = ref.info == 0
    assert np.array_equal(g["info"] != 0, ~ok)
    Ainv = oracle.invert_batched(A[ok]).inverse
    kappa = np.abs(A[ok].astype(np.float64)).sum(2).max(1) * np.abs(Ainv).sum(2).max(1)
    e = np.abs(g["X"][ok] - ref.X[ok]).max(axis=(1, 2)) / np.abs(ref.X[ok]).max(axis=(1, 2))
    assert np.all(e <= np.maximum(2e-4, kappa * EPS)), np.max(e / (kappa * EPS))
    assert np.array_equal(g["sign"][ok], ref.sign[ok].astype(np.int8))
    assert np.all(np.abs(g["logabsdet"][ok] - ref.logabsdet[ok]) <= np.maximum(2e-4, kappa * EPS))


def test_solve_exact_pins(gj, torch):
    """Hadamard systems (ties at every step, every intermediate exact): X = H^T B / 32
    bit-exact for integer B; signed permutations likewise."""
    H = np.stack([synth.hadamard_pd(32, seed=s)[0] for s in range(9)]).astype(np.float32)
    B = np.random.default_rng(7).integers(-4, 5, (9, 32, 3)).astype(np.float32)
    g = solve(gj, torch, H, B, 0.0)
    assert np.array_equal(g["X"], np.einsum("bji,bjk->bik", H, B) / 32)
    rng = np.random.default_rng(8)
    P = np.zeros((5, 32, 32), np.float32)
    for b in range(5):
        P[b, np.arange(32), rng.permutation(32)] = rng.choice([-2.0, 0.5, 4.0], 32)
    Bp = rng.integers(-8, 9, (5, 32, 8)).astype(np.float32)
    g = solve(gj, torch, P, Bp, 0.0)
    ref = oracle.solve_batched(P, Bp, tol=0.0)
    assert np.array_equal(g["X"], ref.X.astype(np.float32))
    assert np.array_equal(g["ipiv"], ref.ipiv)


def test_solve_singular_and_inplace(gj, torch):
    rng = np.random.default_rng(9)
    A = synth.gen_normal_batch(300, 32, seed=60, dtype=np.float32)
    S = rng.choice(300, 20, replace=False)
    for b in S:
        A[b, 5] = A[b, 11]
    A[S[0]] = 0.0
    B = rng.standard_normal((300, 32, 4)).astype(np.float32)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    r = gj.solve_batched(At, Bt, tol=1e-5)
    r2 = gj.solve_batched(At, Bt.clone(), tol=1e-5, out=None)
    Xin = Bt.clone()
    r3 = gj.solve_batched(At, Xin, tol=1e-5, out=Xin)   # X aliases B
    torch.cuda.synchronize()
    assert set(np.nonzero(r.info.cpu().numpy())[0]) == set(S.tolist())
    ok = r.info.cpu().numpy() == 0
    assert torch.equal(r.X[ok], r2.X[ok]) and torch.equal(r.X[ok], Xin[ok])
    assert torch.equal(r3.info, r.info)


@pytest.mark.parametrize("batch", [1, 999, 65536])
def test_det_only_matches_inverse_path(gj, torch, batch):
    A = synth.gen_normal_batch(batch, 32, seed=70, dtype=np.float32)
    if batch > 10:
        A[3, 9] = A[3, 1]   # a singular item
    At = torch.from_numpy(A).cuda()
    r1 = gj.invert_batched(At)
    r2 = gj.det(At)
    torch.cuda.synchronize()
    for k in ("logabsdet", "sign", "det", "ipiv", "info"):
        assert torch.equal(getattr(r1, k), getattr(r2, k)), k


def test_k7_beyond_eight_rhs(gj, torch):
    """fp32 n = 32 with more than 8 right-hand sides runs on K7 (gj_solve.cu), the general
    solve kernel: same oracle rule as K1s."""
    A = synth.gen_c2(batch=3000)
    rng = np.random.default_rng(8)
    B = rng.standard_normal((3000, 32, 12)).astype(np.float32)
    r = gj.solve_batched(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), tol=32 * 2.0 ** -23)
    torch.cuda.synchronize()
    ref = oracle.solve_batched(A, B, tol=32 * 2.0 ** -23)
    ok = ref.info == 0
    Ainv = oracle.invert_batched(A[ok]).inverse
    kappa = np.abs(A[ok].astype(np.float64)).sum(2).max(1) * np.abs(Ainv).sum(2).max(1)
    X = r.X.cpu().numpy()
    e = np.abs(X[ok] - ref.X[ok]).max(axis=(1, 2)) / np.abs(ref.X[ok]).max(axis=(1, 2))
    assert np.all(e <= np.maximum(2e-4, kappa * 2.0 ** -23))

"""GPU parity of the batched multi-RHS solve (K7, gj_solve_batched: Gauss–Jordan on [A | B],
SURVEY.md §8f f4) against the oracle's GJ on [A | B] (oracle.solve_batched)."""
import numpy as np
import pytest

import oracle
import synth
from tests.parity import TIE_GAP, TOL_INV, ipiv_match

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


def run(gj, torch, A, B, tol=None, inplace=False):
    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    Bt = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    r = gj.solve_batched(At, Bt, tol, out=Bt if inplace else None)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in r._asdict().items()}


def eps(dtype):
    return 2.0 ** -23 if dtype == np.float32 else 2.0 ** -52


@pytest.mark.parametrize("m", [1, 3, 8, 32])
@pytest.mark.parametrize("n", [1, 2, 5, 16, 17, 32])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_gaussian_vs_oracle(gj, torch, n, m, dtype):
    rng = np.random.default_rng(700 + 10 * n + m)
    Bt = 519   # several warps' tasks, a ragged last task
    A = synth.gen_normal_batch(Bt, n, seed=700 + n, dtype=dtype)
    B = rng.standard_normal((Bt, n, m)).astype(dtype)
    tol = n * eps(dtype)
    g = run(gj, torch, A, B, tol)
    ref = oracle.solve_batched(A, B, tol=tol)
    ok = ref.info == 0
    assert np.array_equal(g["info"] != 0, ~ok)
    Ainv = oracle.invert_batched(A[ok]).inverse
    kappa = np.abs(A[ok].astype(np.float64)).sum(2).max(1) * np.abs(Ainv).sum(2).max(1)
    e = np.abs(g["X"][ok] - ref.X[ok]).max(axis=(1, 2)) / np.abs(ref.X[ok]).max(axis=(1, 2))
    lim = np.maximum(TOL_INV[dtype], kappa * eps(dtype))
    print(f"n={n} m={m}: max e/lim {np.max(e / lim):.3e}")
    assert np.all(e <= lim)
    for b in np.nonzero(ok)[0]:
        assert ipiv_match(g["ipiv"][b], ref.ipiv[b], ref.gap[b])[0]
    assert np.array_equal(g["sign"][ok], ref.sign[ok].astype(np.int8))
    assert np.all(np.abs(g["logabsdet"][ok] - ref.logabsdet[ok]) <= np.maximum(TOL_INV[dtype], kappa * eps(dtype)))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_paper_matrix_exact(gj, torch, dtype):
    """P:L89-L92's matrix: A^-1 = [[3,-3,1],[-3,5,-2],[1,-2,1]], pivots 1, 2, -1/2 — every
    operation exact, so X = A^-1 B exactly for integer B."""
    A = synth.paper_matrix(dtype)[None]
    B = np.array([[[1, 0, 2], [0, 1, -1], [3, 1, 0]]], dtype)
    Ainv = np.array([[3, -3, 1], [-3, 5, -2], [1, -2, 1]], np.float64)
    g = run(gj, torch, A, B)
    assert np.array_equal(g["X"][0], (Ainv @ B[0].astype(np.float64)).astype(dtype))
    assert list(g["ipiv"][0]) == [1, 3, 3] and g["sign"][0] == 1 and g["logabsdet"][0] == 0.0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_inplace_and_singular(gj, torch, dtype):
    rng = np.random.default_rng(71)
    Bt, n, m = 300, 12, 5
    A = rng.standard_normal((Bt, n, n)).astype(dtype)
    A[::7, 4] = A[::7, 2]                 # duplicated rows: singular items
    B = rng.standard_normal((Bt, n, m)).astype(dtype)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    g1 = run(gj, torch, A, B, tol)
    g2 = run(gj, torch, A, B, tol, inplace=True)
    ref = oracle.solve_batched(A, B, tol=tol)
    assert np.array_equal(g1["info"] != 0, ref.info != 0) and (ref.info != 0).sum() == len(range(0, Bt, 7))
    ok = ref.info == 0
    assert np.array_equal(g1["X"][ok], g2["X"][ok])


def test_identity_rhs_matches_inverse_path(gj, torch):
    """B = I: the solve computes A^-1 — the same quantity as gj_invert_batched, through a
    different kernel; both within the parity bound of the oracle's inverse."""
    A = synth.gen_normal_batch(256, 24, seed=72, dtype=np.float64)
    B = np.broadcast_to(np.eye(24), (256, 24, 24)).copy()
    g = run(gj, torch, A, B)
    inv = gj.invert_batched(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    Xi = inv.inverse.cpu().numpy()
    Xr = oracle.invert_batched(A).inverse
    kappa = np.abs(A).sum(2).max(1) * np.abs(Xr).sum(2).max(1)
    for X in (g["X"], Xi):
        e = np.abs(X - Xr).max(axis=(1, 2)) / np.abs(Xr).max(axis=(1, 2))
        assert np.all(e <= np.maximum(1e-10, kappa * 2.0 ** -52))
    assert np.array_equal(g["ipiv"], inv.ipiv.cpu().numpy())


# ------------------------------------------------------------------ large n (gj_solve, fp64)
def run_single(gj, torch, A, B, tol=None, strided=False):
    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    Bt = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    if strided:   # views with padded rows
        Ap = torch.zeros((A.shape[0], A.shape[1] + 7), dtype=At.dtype, device="cuda")
        Ap[:, :A.shape[1]] = At
        Bp = torch.zeros((B.shape[0], B.shape[1] + 3), dtype=Bt.dtype, device="cuda")
        Bp[:, :B.shape[1]] = Bt
        At, Bt = Ap[:, :A.shape[1]], Bp[:, :B.shape[1]]
    r = gj.solve(At, Bt, tol)
    torch.cuda.synchronize()
    return r.X.cpu().numpy(), int(r.info), int(r.sign), float(r.logabsdet), r.ipiv.cpu().numpy()


@pytest.mark.parametrize("n,m", [(33, 1), (64, 5), (100, 40), (300, 7), (777, 3), (1024, 33)])
def test_large_solve_vs_oracle(gj, torch, n, m):
    A = synth.gen_gaussian(n, seed=900 + n)
    B = np.random.default_rng(n).standard_normal((n, m))
    X, info, sg, lg, ipiv = run_single(gj, torch, A, B, strided=(n % 2 == 1))
    ref = oracle.solve_batched(A, B)
    Ai = oracle.invert(A).inverse[0]
    kappa = np.abs(A).sum(1).max() * np.abs(Ai).sum(1).max()
    e = np.abs(X - ref.X[0]).max() / np.abs(ref.X[0]).max()
    print(f"n={n} m={m}: rel err {e:.3e} kappa {kappa:.3e}")
    assert info == 0
    assert e <= max(1e-10, kappa * 2.0 ** -52)
    assert ipiv_match(ipiv, ref.ipiv[0], ref.gap[0])[0]
    assert sg == ref.sign[0] and abs(lg - ref.logabsdet[0]) <= max(1e-10, kappa * 2.0 ** -52)


def test_large_solve_hadamard_exact(gj, torch):
    """P6-style pin: every pivot a power of two and every value a small dyadic number, so
    X = A^T B / n exactly for an integer B."""
    n = 512
    A = synth.hadamard_pd(n, seed=5)[0]
    B = np.random.default_rng(3).integers(-4, 5, (n, 6)).astype(np.float64)
    X, info, _, lg, _ = run_single(gj, torch, A, B)
    assert info == 0
    assert np.array_equal(X, A.T @ B / n)


def test_large_solve_identity_rhs_matches_invert(gj, torch):
    n = 700
    A = synth.gen_gaussian(n, seed=77)
    X, info, sg, lg, ipiv = run_single(gj, torch, A, np.eye(n))
    r = gj.invert(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(ipiv, r.ipiv.cpu().numpy())
    assert lg == float(r.logabsdet) and sg == int(r.sign)
    Xi = r.inverse.cpu().numpy()
    assert np.abs(X - Xi).max() / np.abs(Xi).max() <= 1e-11


def test_large_solve_singular(gj, torch):
    A = synth.gen_gaussian(200, seed=78)
    A[150] = A[20]
    _, info, sg, lg, _ = run_single(gj, torch, A, np.ones((200, 2)), tol=1e-10)
    ref = oracle.solve_batched(A, np.ones((200, 2)), tol=1e-10)
    assert info == ref.info[0] > 0 and sg == 0 and lg == -np.inf


@pytest.mark.parametrize("n,m", [(33, 2), (65, 1), (300, 40), (1024, 5)])
def test_large_solve_f32_vs_oracle(gj, torch, n, m):
    """fp32 beyond the batched limits: the tcgen05 (3xTF32) blocked path on [A | B]."""
    A = synth.gen_gaussian(n, seed=950 + n).astype(np.float32)
    B = np.random.default_rng(n + 1).standard_normal((n, m)).astype(np.float32)
    X, info, sg, lg, ipiv = run_single(gj, torch, A, B)
    ref = oracle.solve_batched(A, B)
    Ai = oracle.invert(A).inverse[0]
    kappa = np.abs(A.astype(np.float64)).sum(1).max() * np.abs(Ai).sum(1).max()
    e = np.abs(X - ref.X[0]).max() / np.abs(ref.X[0]).max()
    print(f"fp32 n={n} m={m}: rel err {e:.3e} kappa {kappa:.3e}")
    assert info == 0
    assert e <= max(TOL_INV[np.float32], kappa * 2.0 ** -23)
    assert ipiv_match(ipiv, ref.ipiv[0], ref.gap[0])[0]
    assert sg == ref.sign[0]


def test_large_solve_f32_hadamard_exact(gj, torch):
    n = 256
    A = synth.hadamard_pd(n, seed=5)[0].astype(np.float32)
    B = np.random.default_rng(4).integers(-4, 5, (n, 3)).astype(np.float32)
    X, info, _, _, _ = run_single(gj, torch, A, B)
    assert info == 0 and np.array_equal(X, (A.T.astype(np.float64) @ B / n).astype(np.float32))

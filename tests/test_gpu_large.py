"""GPU parity of the large-n blocked path (gj_invert, n > 64: cluster leaf factorisation
+ FP64 tensor-core trailing updates) against the oracle and exact pins."""
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests.parity import TOL_INV, TOL_RES, ipiv_match

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def gj():
    import paper_1401_7962_b200 as g
    return g


def run_single(gj, torch, A, tol=None):
    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    r = gj.invert(At, tol=tol)
    torch.cuda.synchronize()
    return {"inverse": r.inverse.cpu().numpy(), "ipiv": r.ipiv.cpu().numpy(), "logabsdet": float(r.logabsdet),
            "sign": int(r.sign), "info": int(r.info)}


@pytest.mark.parametrize("n", [65, 96, 100, 256, 777, 1024])
def test_gaussian_vs_oracle(gj, torch, n):
    A = synth.gen_gaussian(n, seed=40 + n)
    tol = n * 2.0 ** -52
    g = run_single(gj, torch, A, tol)
    ref = oracle.invert(A, tol=tol)
    X = ref.inverse[0]
    kappa = oracle.kappa_inf(A, X)[0]
    e = np.abs(g["inverse"] - X).max() / np.abs(X).max()
    assert g["info"] == 0
    assert e <= max(TOL_INV[np.float64], kappa * 2.0 ** -52), (e, kappa)
    ok, _ = ipiv_match(g["ipiv"], ref.ipiv[0], ref.gap[0])
    assert ok
    assert g["sign"] == ref.sign[0]
    assert abs(g["logabsdet"] - ref.logabsdet[0]) <= max(1e-10, kappa * 2.0 ** -52)
    assert oracle.residual(A, g["inverse"]) <= max(TOL_RES[np.float64], kappa * 2.0 ** -52)


@pytest.mark.parametrize("n", [128, 1024, 2048])
def test_hadamard_exact(gj, torch, n):
    """P6 at scale: every step an exact tie; exact inverse A^T/n, (n/2) ln n, getrf ipiv."""
    import scipy.linalg
    A, _, _ = synth.hadamard_pd(n, seed=5)
    g = run_single(gj, torch, A)
    assert np.array_equal(g["inverse"], A.T / n)
    assert abs(g["logabsdet"] - 0.5 * n * math.log(n)) <= 1e-12 * n
    _, piv = scipy.linalg.lu_factor(A)
    assert np.array_equal(g["ipiv"], piv + 1)
    s, _ = np.linalg.slogdet(A)
    assert g["sign"] == s


def test_singular_flag(gj, torch):
    A = synth.gen_gaussian(300, seed=7)
    A[123] = A[45]
    g = run_single(gj, torch, A, tol=1e-10)
    ref = oracle.invert(A, tol=1e-10)
    assert ref.info[0] > 0
    assert g["info"] == ref.info[0]
    assert g["sign"] == 0 and g["logabsdet"] == -np.inf


@pytest.mark.parametrize("n", [200, 1000])
def test_det_entry_large(gj, torch, n):
    """gj_det (the trailing update restricted to the columns right of the next panel) takes
    the same pivots and pivot values as gj_invert: identical ipiv, log|det| and sign."""
    A = synth.gen_gaussian(n, seed=8)
    At = torch.from_numpy(A).cuda()
    r1 = gj.invert(At)
    r2 = gj.det(At)
    torch.cuda.synchronize()
    assert torch.equal(r1.ipiv, r2.ipiv)
    assert float(r1.logabsdet) == float(r2.logabsdet)
    assert int(r1.sign) == int(r2.sign)
    s, ld = np.linalg.slogdet(A)
    assert int(r2.sign) == int(s)
    assert abs(float(r2.logabsdet) - ld) <= 1e-9 * n
    if n <= 200:
        assert abs(float(r2.det) - s * math.exp(ld)) <= 1e-10 * math.exp(ld)


def test_strided_large(gj, torch):
    base = synth.gen_gaussian(300, seed=9)
    big = torch.from_numpy(base).cuda()
    sub = big[:200, :200]
    r = gj.invert(sub)
    torch.cuda.synchronize()
    ref = oracle.invert(base[:200, :200].copy())
    e = np.abs(r.inverse.cpu().numpy() - ref.inverse[0]).max() / np.abs(ref.inverse[0]).max()
    assert e <= TOL_INV[np.float64]


@pytest.mark.parametrize("fname", sorted(f for f in os.listdir(GOLD) if f.startswith("c4_oracle_ref")) or ["none"])
def test_c4_full_vs_stored_oracle(gj, torch, fname):
    """C4 at full size against the oracle's stored outputs (tools/make_c4_reference.py)."""
    if fname == "none":
        pytest.skip("no stored C4 oracle reference")
    ref = np.load(os.path.join(GOLD, fname))
    n, seed = int(ref["n"]), int(ref["seed"])
    A = synth.gen_gaussian(n, seed)
    g = run_single(gj, torch, A, tol=n * 2.0 ** -52)
    assert g["info"] == 0
    ok, _ = ipiv_match(g["ipiv"], ref["ipiv"], ref["gap"])
    assert ok
    kappa = float(ref["kappa_inf"])
    Xr = ref["inv_rows"]
    e = np.abs(g["inverse"][ref["rows"]] - Xr).max() / np.abs(Xr).max()
    print(f"C4 sampled-row rel err {e:.3e}, kappa_inf {kappa:.3e}")
    assert e <= max(TOL_INV[np.float64], kappa * 2.0 ** -52)
    assert g["sign"] == int(ref["sign"])
    assert abs(g["logabsdet"] - float(ref["logabsdet"])) <= max(1e-10, kappa * 2.0 ** -52)
    res = oracle.residual(A, g["inverse"], rows=ref["rows"])
    assert res <= TOL_RES[np.float64]


@pytest.mark.parametrize("dtype,eps_bit", [(np.float64, 2.0 ** -21), (np.float64, 2.0 ** -44), (np.float32, 2.0 ** -20)])
def test_near_tie_exact_max_large(gj, torch, dtype, eps_bit):
    """The cluster argmax of the panel kernel orders candidates by every bit (see the batched
    test of the same name): the true maximum sits at the last row."""
    n = 300
    rng = np.random.default_rng(3)
    A = rng.uniform(-0.5, 0.5, (n, n))
    A[:, 0] = 0.25
    A[0, 0] = 1.0
    A[n - 1, 0] = -(1.0 + eps_bit)
    A = A.astype(dtype)
    r = gj.invert(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    assert int(r.ipiv[0]) == n

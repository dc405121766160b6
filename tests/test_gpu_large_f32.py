"""GPU parity of the fp32 large-n path (gj_invert, dt = GJ_F32, n > 64: the fp32 panel
kernel + the tcgen05 TF32 trailing update with a 3xTF32 split) against
the oracle (long double on the same fp32 input) and the exact Hadamard pin."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.parity import TOL_INV, ipiv_match

pytestmark = pytest.mark.gpu
EPS32 = 2.0 ** -23


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def gj():
    import paper_1401_7962_b200 as g
    return g


def run(gj, torch, A, tol=None):
    r = gj.invert(torch.from_numpy(np.ascontiguousarray(A)).cuda(), tol=tol)
    torch.cuda.synchronize()
    return (r.inverse.cpu().numpy(), float(r.logabsdet), int(r.sign), int(r.info), r.ipiv.cpu().numpy())


@pytest.mark.parametrize("n", [65, 100, 256, 777, 1024, 2048])
def test_f32_gaussian_vs_oracle(gj, torch, n):
    A = synth.gen_gaussian(n, seed=80 + n).astype(np.float32)
    tol = n * EPS32
    X, lg, sg, info, ipiv = run(gj, torch, A, tol)
    ref = oracle.invert(A, tol=tol)
    Xr = ref.inverse[0]
    kappa = oracle.kappa_inf(A.astype(np.float64), Xr)[0]
    e = np.abs(X - Xr).max() / np.abs(Xr).max()
    print(f"n={n} rel err {e:.3e} kappa {kappa:.3e} e/(kappa eps32) {e / (kappa * EPS32):.3e}")
    assert info == 0
    assert e <= max(TOL_INV[np.float32], kappa * EPS32), (e, kappa)
    ok, _ = ipiv_match(ipiv, ref.ipiv[0], ref.gap[0])
    assert ok
    assert sg == ref.sign[0]
    assert abs(lg - ref.logabsdet[0]) <= max(2e-4, kappa * EPS32)


@pytest.mark.parametrize("n", [128, 1024])
def test_f32_hadamard_exact(gj, torch, n):
    import scipy.linalg
    A = synth.hadamard_pd(n, seed=5)[0].astype(np.float32)
    X, lg, sg, info, ipiv = run(gj, torch, A)
    assert np.array_equal(X, A.T / n)
    assert abs(lg - 0.5 * n * math.log(n)) <= 1e-9 * n
    _, piv = scipy.linalg.lu_factor(A.astype(np.float64))
    assert np.array_equal(ipiv, piv + 1)


def test_f32_diag_dominant_flat(gj, torch):
    """Well conditioned (kappa ~ 1): the flat fp32 bound must hold — measures the 3xTF32
    trailing update's accuracy directly."""
    n = 4096
    rng = np.random.default_rng(91)
    A = (rng.uniform(-1, 1, (n, n)) + 2 * math.sqrt(n) * np.eye(n)).astype(np.float32)
    X, lg, sg, info, ipiv = run(gj, torch, A)
    Xr = np.linalg.inv(A.astype(np.float64))
    e = np.abs(X - Xr).max() / np.abs(Xr).max()
    print(f"diag-dominant n={n}: rel err {e:.3e}")
    assert e <= 1e-5


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_large_repeatable(gj, torch, dtype):
    """Bitwise-identical results over repeated calls at n = 8192 (a 16-CTA cluster of 512
    rows each): guards the leaf kernel's asynchronous DSMEM exchange (a source slot rewritten
    before a peer's bulk copy read it showed up as run-to-run pivot differences)."""
    A = torch.from_numpy(synth.gen_gaussian(8192, seed=3).astype(dtype)).cuda()
    runs = []
    for _ in range(4):
        r = gj.invert(A)
        torch.cuda.synchronize()
        runs.append((r.ipiv.clone(), r.inverse.clone(), float(r.logabsdet)))
    d = gj.det(A)
    torch.cuda.synchronize()
    for ip, X, lg in runs[1:]:
        assert torch.equal(ip, runs[0][0])
        assert torch.equal(X, runs[0][1])
        assert lg == runs[0][2]
    assert float(d.logabsdet) == runs[0][2]


GOLD = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


@pytest.mark.parametrize("fname", sorted(f for f in __import__("os").listdir(GOLD) if f.startswith("f1_oracle_ref"))
                         or ["none"])
def test_f1_full_vs_stored_oracle(gj, torch, fname):
    """f1 at the size bench.py times (fp32 n = 8192) against the oracle's stored outputs on the
    same fp32 input (tools/make_c4_reference.py 8192 3 f32: long-double GJ on [A | I]): the
    pivot sequence (R3; a first divergence only at an oracle gap inside reading G26's
    n u32 band), 64 sampled inverse rows within the kappa rule (R1), log|det| and sign, and
    the residual of the sampled rows (R2)."""
    import os
    from tests.parity import TOL_RES, first_divergence_gap, tie_gap
    if fname == "none":
        pytest.skip("no stored f1 oracle reference")
    ref = np.load(os.path.join(GOLD, fname))
    n, seed = int(ref["n"]), int(ref["seed"])
    A = synth.gen_gaussian(n, seed).astype(np.float32)
    X, lg, sg, info, ipiv = run(gj, torch, A, tol=n * EPS32)
    assert info == 0
    ok, exempt = ipiv_match(ipiv, ref["ipiv"], ref["gap"], thr=tie_gap(np.float32, n))
    print(f"f1 n={n}: first pivot divergence at oracle gap {first_divergence_gap(ipiv, ref['ipiv'], ref['gap'])}")
    assert ok
    kappa = float(ref["kappa_inf"])
    Xr = ref["inv_rows"]
    e = np.abs(X[ref["rows"]] - Xr).max() / np.abs(Xr).max()
    print(f"f1 sampled-row rel err {e:.3e}, kappa_inf {kappa:.3e}, e/(kappa eps32) {e / (kappa * EPS32):.3e}")
    assert e <= max(TOL_INV[np.float32], kappa * EPS32)
    assert sg == int(ref["sign"])
    assert abs(lg - float(ref["logabsdet"])) <= max(2e-4, kappa * EPS32)
    res = oracle.residual(A.astype(np.float64), X.astype(np.float64), rows=ref["rows"])
    assert res <= max(TOL_RES[np.float32], kappa * EPS32)

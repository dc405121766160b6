"""GPU parity of the full-pivoting batched path (K6, gj_invert_batched_full; SURVEY.md §8f
f2, Obs. 2–3 PAPER.md L59–L60) against the full-pivoting oracle
(``oracle.invert_full_batched``), rules R1–R8 with the row AND column swap sequences."""
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


def run(gj, torch, A, tol=None, inverse=True):
    r = gj.invert_batched_full(torch.from_numpy(np.ascontiguousarray(A)).cuda(), tol=tol, inverse=inverse)
    torch.cuda.synchronize()
    return {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}


def eps(dtype):
    return 2.0 ** -23 if dtype == np.float32 else 2.0 ** -52


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 16, 17, 24, 31, 32])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_gaussian_vs_oracle(gj, torch, n, dtype):
    B = 1037   # several warps' worth of tasks and a ragged last task
    A = synth.gen_normal_batch(B, n, seed=300 + n, dtype=dtype)
    tol = n * eps(dtype)
    g = run(gj, torch, A, tol)
    ref = oracle.invert_full_batched(A, tol=tol)
    rep = compare(A, g, ref, dtype, tol)
    print(rep.summary())
    assert_report(rep)


@pytest.mark.parametrize("n", [4, 16, 32])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_hadamard(gj, torch, n, dtype):
    """Sylvester–Hadamard A = P H D: exact ties at most steps, so the G23 rule decides the
    pivots.  Where every pivot of the oracle is a power of two the whole elimination is
    exact in any precision and the GPU must match bit for bit (inverse A^T / n, ipiv,
    jpiv); otherwise (a pivot like 3/2 makes later values inexact, and rounding then
    decides the ties) rules R1-R8 apply."""
    A = np.stack([synth.hadamard_pd(n, seed=s)[0] for s in range(16)]).astype(dtype)
    g = run(gj, torch, A)
    ref = oracle.invert_full_batched(A)
    pv = np.abs(ref.pivots)
    exact = np.all(np.log2(pv) == np.round(np.log2(pv)), axis=1)
    assert exact.sum() >= 2
    e = np.nonzero(exact)[0]
    assert np.array_equal(g["inverse"][e], np.transpose(A[e], (0, 2, 1)) / n)
    assert np.array_equal(g["ipiv"][e], ref.ipiv[e])
    assert np.array_equal(g["jpiv"][e], ref.jpiv[e])
    assert np.array_equal(g["sign"], ref.sign.astype(np.int8))
    rep = compare(A, g, ref, dtype, n * eps(dtype))
    print(f"exact items {exact.sum()}/16; " + rep.summary())
    assert_report(rep)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_permutations_bit_exact(gj, torch, dtype):
    from oracle import exact
    perms = list(synth.all_permutations(5))
    A = np.stack([synth.permutation_matrix(p) for p in perms]).astype(dtype)
    g = run(gj, torch, A)
    ref = oracle.invert_full_batched(A)
    assert np.array_equal(g["inverse"], np.transpose(A, (0, 2, 1)))
    assert np.array_equal(g["ipiv"], ref.ipiv) and np.array_equal(g["jpiv"], ref.jpiv)
    assert np.array_equal(g["sign"], np.array([exact.permutation_sign(p) for p in perms], np.int8))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_integer_ties_and_singular(gj, torch, dtype):
    """Small integers: exact ties are frequent (R3 exempts only real near-ties), and a share
    of the items is singular (duplicated rows / zero columns)."""
    rng = np.random.default_rng(31)
    B, n = 2000, 7
    A = rng.integers(-3, 4, (B, n, n)).astype(dtype)
    A[::17, 3] = A[::17, 1]
    A[5::23, :, 2] = 0
    tol = 1e-5 if dtype == np.float32 else 1e-12
    g = run(gj, torch, A, tol)
    ref = oracle.invert_full_batched(A, tol=tol)
    assert ref.info.astype(bool).sum() > 100
    rep = compare(A, g, ref, dtype, tol)
    print(rep.summary())
    assert_report(rep)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_det_only_same_outputs(gj, torch, dtype):
    A = synth.gen_normal_batch(300, 20, seed=7, dtype=dtype)
    g1 = run(gj, torch, A)
    g2 = run(gj, torch, A, inverse=False)
    assert g2["inverse"] is None
    for k in ("logabsdet", "sign", "det", "ipiv", "jpiv", "info"):
        assert np.array_equal(g1[k], g2[k]), k

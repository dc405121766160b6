"""GPU parity of the batched path (K1, n <= 32) against the oracle, through the C-ABI
binding.  Rules R1–R8 (tests/parity.py)."""
import numpy as np
import pytest

import oracle
import synth
from tests.parity import TOL_INV, TOL_RES, assert_report, compare

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


def run_gpu(gj, torch, A, tol=None, inplace=False):
    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    r = gj.invert_batched(At, tol=tol, out=At if inplace else None)
    torch.cuda.synchronize()
    return {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}


def default_tol(dtype, n):
    return n * (2.0 ** -23 if dtype == np.float32 else 2.0 ** -52)


# ------------------------------------------------------------------ exact pins (R8)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_paper_matrix_bit_exact(gj, torch, dtype):
    A = synth.paper_matrix(dtype)[None]
    g = run_gpu(gj, torch, A)
    assert np.array_equal(g["inverse"][0], np.array([[3, -3, 1], [-3, 5, -2], [1, -2, 1]], dtype))
    assert list(g["ipiv"][0]) == [1, 3, 3]
    assert g["det"][0] == 1.0 and g["sign"][0] == 1 and g["logabsdet"][0] == 0.0 and g["info"][0] == 0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_permutation_matrices_bit_exact(gj, torch, n, dtype):
    from oracle import exact
    perms = list(synth.all_permutations(n))
    A = np.stack([synth.permutation_matrix(p) for p in perms]).astype(dtype)
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A)
    assert np.array_equal(g["inverse"], np.transpose(A, (0, 2, 1)))
    assert np.array_equal(g["ipiv"], ref.ipiv)
    assert np.array_equal(g["sign"], np.array([exact.permutation_sign(p) for p in perms], np.int8))
    assert np.all(g["det"] == g["sign"])


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_hadamard_bit_exact(gj, torch, n, dtype):
    """P6: every step an exact tie (tie-break G3 at every step), every value dyadic."""
    A = np.stack([synth.hadamard_pd(n, seed=5 + s)[0] for s in range(40)]).astype(dtype)
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A)
    assert np.array_equal(g["inverse"], (np.transpose(A, (0, 2, 1)) / n).astype(dtype))
    assert np.array_equal(g["ipiv"], ref.ipiv)
    assert np.array_equal(g["sign"].astype(np.int32), ref.sign)
    np.testing.assert_allclose(g["logabsdet"], 0.5 * n * np.log(n), rtol=1e-14)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_signed_perm_pow2_bit_exact(gj, torch, dtype):
    mats = []
    for s in range(20):
        A, _, _ = synth.signed_perm_pow2(32, seed=s)
        mats.append(A)
    A = np.stack(mats).astype(dtype)
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A)
    assert np.array_equal(g["inverse"], ref.inverse.astype(dtype))


# ------------------------------------------------------------------ C1 (configs[0]) full size
def test_c1_full(gj, torch):
    A = synth.gen_c1()
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A, tol=default_tol(np.float64, 16))
    # item 0 = blockdiag(P3, I13): bit exact (P1)
    exp = np.eye(16)
    exp[:3, :3] = [[3, -3, 1], [-3, 5, -2], [1, -2, 1]]
    assert np.array_equal(g["inverse"][0], exp)
    assert list(g["ipiv"][0]) == [1, 3, 3] + list(range(4, 17))
    assert g["det"][0] == 1.0
    rep = compare(A, g, ref, np.float64, default_tol(np.float64, 16), check_det=True, flat_only=True)
    assert_report(rep, flat_only=True)
    res = oracle.residual_batched(A, g["inverse"])
    assert res.max() <= TOL_RES[np.float64]


# ------------------------------------------------------------------ C2 (configs[1])
def test_c2_prefix(gj, torch):
    """First 32768 items of the seed-1 stream (identical to the full config's prefix)."""
    A = synth.gen_c2(batch=32768)
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A, tol=default_tol(np.float32, 32))
    rep = compare(A, g, ref, np.float32, default_tol(np.float32, 32))
    print(rep.summary())
    assert_report(rep)
    res = oracle.residual_batched(A, g["inverse"])
    kappa = oracle.kappa_inf(A, ref.inverse)
    reg = ref.info == 0
    lim = np.maximum(TOL_RES[np.float32], kappa * 2.0 ** -23)
    assert np.all(res[reg] <= lim[reg])


# ------------------------------------------------------------------ C3 (configs[2])
def test_c3_prefix(gj, torch):
    """C3 recipe (reading G15) at batch 8192 with 1% duplicated-row singular items, tol 1e-10:
    flat fp64 tolerances (well-conditioned), exact singular-flag agreement (R7)."""
    A, S = synth.gen_c3(batch=8192, return_singular=True)
    g = run_gpu(gj, torch, A, tol=synth.C3_TOL)
    ref = oracle.invert_batched(A, tol=synth.C3_TOL)
    assert np.array_equal(np.nonzero(ref.info)[0], S)
    assert np.array_equal(np.nonzero(g["info"])[0], S)
    rep = compare(A, g, ref, np.float64, synth.C3_TOL, flat_only=True)
    print(rep.summary())
    assert_report(rep, flat_only=True)
    reg = ref.info == 0
    res = oracle.residual_batched(A[reg][:2000], g["inverse"][reg][:2000])
    assert res.max() <= TOL_RES[np.float64]


# ------------------------------------------------------------------ ragged shapes
@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 9, 12, 13, 17, 24, 31, 32, 33, 40, 47, 63, 64])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_ragged_sizes(gj, torch, n, dtype):
    B = 517  # not a multiple of any group count: ragged tail
    A = synth.gen_normal_batch(B, n, seed=100 + n, dtype=dtype)
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A, tol=default_tol(dtype, n))
    rep = compare(A, g, ref, dtype, default_tol(dtype, n))
    assert_report(rep)


def test_empty_batch(gj, torch):
    A = torch.empty((0, 8, 8), dtype=torch.float32, device="cuda")
    r = gj.invert_batched(A)
    assert r.inverse.shape == (0, 8, 8)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [32, 64])
def test_in_place_equals_out_of_place(gj, torch, dtype, n):
    A = synth.gen_normal_batch(300, n, seed=5, dtype=dtype)
    g1 = run_gpu(gj, torch, A)
    g2 = run_gpu(gj, torch, A, inplace=True)
    for k in ("inverse", "ipiv", "logabsdet", "sign", "info"):
        assert np.array_equal(g1[k], g2[k])


def test_batch_order_invariance(gj, torch):
    A = synth.gen_normal_batch(999, 16, seed=6, dtype=np.float32)
    perm = np.random.default_rng(0).permutation(999)
    g1 = run_gpu(gj, torch, A)
    g2 = run_gpu(gj, torch, A[perm])
    assert np.array_equal(g2["inverse"], g1["inverse"][perm])
    assert np.array_equal(g2["ipiv"], g1["ipiv"][perm])


# ------------------------------------------------------------------ singular items (Obs. 2)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_singular_flags(gj, torch, dtype):
    rng = np.random.default_rng(8)
    B, n = 256, 12
    A = rng.standard_normal((B, n, n)).astype(dtype)
    sing = rng.choice(B, 40, replace=False)
    for b in sing:
        i, j = rng.choice(n, 2, replace=False)
        A[b, j] = A[b, i]
    A[sing[0]] = 0.0                       # all-zero matrix -> singular at step 1
    tol = 1e-10 if dtype == np.float64 else 1e-5
    g = run_gpu(gj, torch, A, tol=tol)
    ref = oracle.invert_batched(A, tol=tol)
    assert g["info"][sing[0]] == 1
    rep = compare(A, g, ref, dtype, tol)
    assert_report(rep)
    flagged = np.nonzero(g["info"])[0]
    assert set(flagged) == set(sing.tolist())
    assert np.all(g["sign"][flagged] == 0) and np.all(g["det"][flagged] == 0)
    assert np.all(np.isneginf(g["logabsdet"][flagged]))


def test_zero_pivot_not_singular(gj, torch):
    A = np.array([[[0.0, 1.0], [1.0, 0.0]]])
    g = run_gpu(gj, torch, A, tol=0.0)
    assert g["info"][0] == 0 and np.array_equal(g["inverse"][0], A[0]) and g["det"][0] == -1.0


# ------------------------------------------------------------------ other entry points
@pytest.mark.parametrize("n,dtype", [(20, np.float64), (64, np.float64), (32, np.float32), (48, np.float32)])
def test_det_entry_matches_invert(gj, torch, n, dtype):
    """gj_det (Ainv = NULL) — the det-only kernels (K1s for fp32 n = 32, K2f skipping the
    compact D columns for fp64 n = 64) give bitwise the inverting path's pivots and dets."""
    A = synth.gen_normal_batch(700, n, seed=9, dtype=dtype)
    A[5, 3] = A[5, 1]   # a singular item
    At = torch.from_numpy(A).cuda()
    r1 = gj.invert_batched(At)
    r2 = gj.det(At)
    torch.cuda.synchronize()
    for k in ("logabsdet", "sign", "det", "ipiv", "info"):
        assert torch.equal(getattr(r1, k), getattr(r2, k)), k


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_host_entry_matches_device(gj, torch, dtype):
    A = synth.gen_normal_batch(5000, 32, seed=11, dtype=dtype)
    g = run_gpu(gj, torch, A)
    X = np.empty_like(A)
    ipiv = np.empty((5000, 32), np.int32)
    lg = np.empty(5000)
    sg = np.empty(5000, np.int8)
    info = np.empty(5000, np.int32)
    gj.invert_batched_host(A, out=X, ipiv=ipiv, logabsdet=lg, sign=sg, info=info, chunk=1234)
    assert np.array_equal(X, g["inverse"]) and np.array_equal(ipiv, g["ipiv"])
    assert np.array_equal(lg, g["logabsdet"]) and np.array_equal(sg, g["sign"])


def test_single_strided(gj, torch):
    base = synth.gen_normal_batch(1, 40, seed=3, dtype=np.float64)[0]
    big = torch.from_numpy(base).cuda()
    sub = big[:24, :24]           # lda = 40
    r = gj.invert(sub)
    torch.cuda.synchronize()
    ref = oracle.invert_batched(base[:24, :24].copy())
    e = np.abs(r.inverse.cpu().numpy() - ref.inverse[0]).max() / np.abs(ref.inverse[0]).max()
    assert e <= TOL_INV[np.float64]
    assert np.array_equal(r.ipiv.cpu().numpy(), ref.ipiv[0])


@pytest.mark.parametrize("n", [8, 32, 48, 64])
@pytest.mark.parametrize("dtype,eps_bit", [(np.float32, 2.0 ** -20), (np.float64, 2.0 ** -21), (np.float64, 2.0 ** -44)])
def test_near_tie_exact_max(gj, torch, n, dtype, eps_bit):
    """Obs. 3 asks for THE maximum |a_ik|: candidates that differ only in the last mantissa
    bits (below the R3 1e-6 tie band, so the general rule would excuse a wrong pick) must
    still be ordered exactly — the key comparison may not drop any bit of the value."""
    # fp64: 2^-21 is bit 31 of the low 32-bit key word, 2^-44 bit 8
    rng = np.random.default_rng(n)
    A = rng.uniform(-0.5, 0.5, (n, n))
    A[:, 0] = 0.25
    A[0, 0] = 1.0
    A[n - 1, 0] = -(1.0 + eps_bit)          # the true maximum, at the last position
    A = A.astype(dtype)[None]
    g = run_gpu(gj, torch, A)
    ref = oracle.invert_batched(A)
    assert ref.ipiv[0, 0] == n and g["ipiv"][0, 0] == n

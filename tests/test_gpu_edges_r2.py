"""Edge cases added in round 2:

* an 8-byte-aligned (not 16-byte-aligned) fp64 n = 64 batch — K2f's 16-byte vector loads
  cannot take it, the launcher must route it to the generic K2 (same oracle rules), not fault;
* the largest order the large-n path accepts, n = GJ_LARGE_MAX_N = 65536, through the
  C-ABI gj_invert: the Sylvester-Hadamard pin P6 (every pivot step an exact tie; the exact
  inverse is A^T / n), built on the device;
* the binding refuses outputs whose shape / dtype / device / layout differ from what the
  library writes (no raw-pointer writes out of bounds)."""
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


def test_misaligned_fp64_n64_batch(gj, torch):
    A = synth.gen_c3(batch=300, seed=21)
    flat = torch.empty(A.size + 1, dtype=torch.float64, device="cuda")
    flat[1:] = torch.from_numpy(A.ravel()).cuda()
    Am = flat[1:].view(A.shape)                       # 8-byte aligned, not 16
    assert Am.data_ptr() % 16 == 8
    out_flat = torch.empty_like(flat)
    Xm = out_flat[1:].view(A.shape)
    r = gj.invert_batched(Am, tol=synth.C3_TOL, out=Xm)
    torch.cuda.synchronize()
    g = {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}
    ref = oracle.invert_batched(A, tol=synth.C3_TOL)
    rep = compare(A, g, ref, np.float64, synth.C3_TOL, flat_only=True)
    assert_report(rep, flat_only=True)
    # and the aligned run of the same items agrees to the flat bound too
    ra = gj.invert_batched(torch.from_numpy(A).cuda(), tol=synth.C3_TOL)
    torch.cuda.synchronize()
    assert np.array_equal(ra.info.cpu().numpy(), g["info"])


def _hadamard_pd_device(torch, n, seed=5):
    """A = P H D on the device (H_ij = (-1)^popcount(i & j)); the exact inverse is D H^T P^T / n."""
    rng = np.random.default_rng(seed)
    perm = torch.from_numpy(rng.permutation(n)).cuda()
    signs = torch.from_numpy(rng.choice(np.array([-1.0, 1.0]), n)).cuda()
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    j = torch.arange(n, device="cuda", dtype=torch.int64)
    for r0 in range(0, n, 1024):
        i = perm[r0:r0 + 1024].view(-1, 1)
        v = i & j.view(1, -1)
        for sh in (16, 8, 4, 2, 1):          # parity of popcount(i & j), indices < 2^32
            v ^= v >> sh
        A[r0:r0 + 1024] = (1.0 - 2.0 * (v & 1).to(torch.float64)) * signs.view(1, -1)
        del v
    return A


def test_largest_order_hadamard_exact(gj, torch):
    """n = 65536 = GJ_LARGE_MAX_N through gj_invert: bit-exact inverse A^T / n (P6)."""
    n = 65536
    free, _ = torch.cuda.mem_get_info()
    if free < 120 * 2 ** 30:
        pytest.skip("needs ~120 GiB of device memory (B200: 180 GB)")
    A = _hadamard_pd_device(torch, n)
    r = gj.invert(A)
    torch.cuda.synchronize()
    assert int(r.info) == 0
    X = r.inverse
    del r
    # exact: X == A^T / n, compared block by block
    for c0 in range(0, n, 4096):
        assert torch.equal(X[:, c0:c0 + 4096], A[c0:c0 + 4096, :].t() / n), c0


def test_binding_rejects_mismatched_outputs(gj, torch):
    A = torch.from_numpy(synth.gen_c2(batch=8)).cuda()
    with pytest.raises(ValueError):
        gj.invert_batched(A, out=torch.empty((8, 32, 31), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        gj.invert_batched(A, out=torch.empty((8, 32, 32), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        gj.invert_batched(A, out=torch.empty((8, 32, 32), dtype=torch.float32))
    with pytest.raises(ValueError):
        gj.invert_batched(A, out=torch.empty((8, 32, 64), dtype=torch.float32, device="cuda")[:, :, ::2])
    with pytest.raises(ValueError):
        gj.det(torch.empty((4, 64, 32), dtype=torch.float32, device="cuda").transpose(1, 2))
    with pytest.raises(ValueError):
        gj.det(torch.empty((4, 3, 5), dtype=torch.float32, device="cuda"))
    B = torch.empty((8, 32, 2), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        gj.solve_batched(A, B, out=torch.empty((8, 32, 3), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        gj.invert(torch.empty((300, 300), dtype=torch.float64, device="cuda"),
                  out=torch.empty((300, 299), dtype=torch.float64, device="cuda"))
    Ah = synth.gen_c2(batch=4)
    with pytest.raises(ValueError):
        gj.invert_batched_host(Ah, out=np.empty((4, 32, 32), np.float64))
    with pytest.raises(ValueError):
        gj.invert_batched_host(Ah, out=np.empty((3, 32, 32), np.float32))
    with pytest.raises(TypeError):
        gj.invert_batched_host(Ah.astype(np.float16), out=np.empty((4, 32, 32), np.float16))

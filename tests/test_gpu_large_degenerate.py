"""Degenerate single large matrices through gj_invert / gj_det / gj_solve, both dtypes:
all-zero, a zero column, a zero first row, a duplicated row (NaN rows after the zero pivot
in the cluster panel kernel), identity.  Nothing may fault; every singular one is flagged
by all three entries, the identity is not and inverts exactly."""
import numpy as np
import pytest

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


@pytest.mark.parametrize("n", [65, 300, 1000])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("case", ["zero", "zerocol", "zerorow0", "duprow", "identity"])
def test_large_degenerate(gj, torch, n, dtype, case):
    rng = np.random.default_rng(n)
    if case == "zero":
        M = np.zeros((n, n))
    elif case == "identity":
        M = np.eye(n)
    else:
        M = rng.standard_normal((n, n))
        if case == "zerocol":
            M[:, 3] = 0.0
        elif case == "zerorow0":
            M[0] = 0.0
        else:
            M[7] = M[2]
    At = torch.from_numpy(M.astype(dtype)).cuda()
    r = gj.invert(At)
    d = gj.det(At)
    s = gj.solve(At, torch.ones((n, 2), dtype=At.dtype, device="cuda"))
    torch.cuda.synchronize()
    flags = [int(x.info.item()) for x in (r, d, s)]
    if case == "identity":
        assert flags == [0, 0, 0]
        assert np.array_equal(r.inverse.cpu().numpy(), np.eye(n, dtype=dtype))
        assert np.array_equal(s.X.cpu().numpy(), np.ones((n, 2), dtype))
    else:
        assert all(f != 0 for f in flags), flags
        assert int(r.sign.item()) == 0 and np.isneginf(float(r.logabsdet.item()))

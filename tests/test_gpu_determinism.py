"""Run-to-run bitwise repeatability of every batched kernel family (compute-sanitizer is not
available on this pool; a race in shared memory, TMEM or the pipelines shows up as results
that change between identical launches — as the large-n leaf race did)."""
import numpy as np
import pytest

import synth

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


def same(runs):
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            if a is None:
                continue
            assert np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("n,dtype", [(32, np.float32), (16, np.float64), (48, np.float32), (64, np.float64),
                                     (32, np.float64)])
def test_batched_repeatable(gj, torch, n, dtype):
    A = torch.from_numpy(synth.gen_normal_batch(60_001, n, seed=n, dtype=dtype)).cuda()
    runs = []
    for _ in range(3):
        r = gj.invert_batched(A)
        torch.cuda.synchronize()
        runs.append([v.cpu().numpy() for v in (r.inverse, r.ipiv, r.logabsdet, r.sign, r.info)])
    same(runs)


def test_next_rows_repeatable(gj, torch):
    A = torch.from_numpy(synth.gen_normal_batch(40_003, 32, seed=9, dtype=np.float32)).cuda()
    B = torch.randn(40_003, 32, 4, device="cuda")
    for f in (lambda: gj.invert_batched_full(A), lambda: gj.invert_batched_pivoting(A, "none"),
              lambda: gj.solve_batched(A, B)):
        runs = []
        for _ in range(3):
            r = f()
            torch.cuda.synchronize()
            runs.append([v.cpu().numpy() for v in r])
        same(runs)

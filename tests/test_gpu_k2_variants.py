"""The fp64 n = 64 kernels that are not the default (GJ_K2_VARIANT, read once per process,
so each runs in a subprocess): K2d (2, the matrix in four warps' registers) and K2b (1,
column-split) — C3 prefix with its singular flags, exact pins, against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_1401_7962_b200 as gj, oracle, synth
from tests.parity import compare, assert_report
A, S = synth.gen_c3(batch=8192, return_singular=True)
r = gj.invert_batched(torch.from_numpy(A).cuda(), tol=synth.C3_TOL)
torch.cuda.synchronize()
g = {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}
assert np.array_equal(np.nonzero(g["info"])[0], S)
idx = np.unique(np.concatenate([np.arange(0, 8192, 41), S]))
ref = oracle.invert_batched(A[idx], tol=synth.C3_TOL)
rep = compare(A[idx], {k: (None if v is None else v[idx]) for k, v in g.items()}, ref, np.float64, synth.C3_TOL,
              flat_only=True)
print(rep.summary()); assert_report(rep, flat_only=True)
H = np.stack([synth.hadamard_pd(64, seed=s)[0] for s in range(5)])
r = gj.invert_batched(torch.from_numpy(H).cuda())
torch.cuda.synchronize()
assert np.array_equal(r.inverse.cpu().numpy(), np.transpose(H, (0, 2, 1)) / 64)
print("variant ok")
'''


@pytest.mark.parametrize("variant", ["1", "2"])
def test_k2_variant(variant):
    env = dict(os.environ, GJ_K2_VARIANT=variant)
    p = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    print(p.stdout[-2000:], p.stderr[-2000:])
    assert p.returncode == 0 and "variant ok" in p.stdout

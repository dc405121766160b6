"""The experimental tensor-core variant of the fp32 n = 32 batched path (K1t,
gj_batched_tc.cu, selected by GJ_K1_TC=1): parity with the oracle on the same rules as K1b,
including a ragged batch (padding matrices in the last task), singular items (which must
not disturb the other matrices of their task through the shared product) and exact pins.
Run in a subprocess because the switch is read once per process."""
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
tol = 32 * 2.0 ** -23
def run(A, tol=tol):
    r = gj.invert_batched(torch.from_numpy(A).cuda(), tol=tol)
    torch.cuda.synchronize()
    return {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}
# ragged Gaussian batch
A = synth.gen_normal_batch(4097, 32, seed=21, dtype=np.float32)
g = run(A); ref = oracle.invert_batched(A, tol=tol)
rep = compare(A, g, ref, np.float32, tol); print(rep.summary()); assert_report(rep)
# singular items mixed in (duplicated rows, an all-zero matrix)
rng = np.random.default_rng(3)
B = synth.gen_normal_batch(1000, 32, seed=22, dtype=np.float32)
S = rng.choice(1000, 60, replace=False)
for b in S: B[b, 7] = B[b, 3]
B[S[0]] = 0.0
g = run(B, 1e-5); ref = oracle.invert_batched(B, tol=1e-5)
rep = compare(B, g, ref, np.float32, 1e-5); print(rep.summary()); assert_report(rep)
assert set(np.nonzero(g["info"])[0]) == set(S.tolist())
# exact pins: Hadamard (ties at every step)
H = np.stack([synth.hadamard_pd(32, seed=s)[0] for s in range(12)]).astype(np.float32)
g = run(H)
assert np.array_equal(g["inverse"], np.transpose(H, (0, 2, 1)) / 32)
print("K1t ok")
'''


def test_k1t_parity():
    env = dict(os.environ, GJ_K1_TC="1", GJ_TC_DEBUG="1")
    code = SCRIPT.replace("ROOT", repr(ROOT))
    p = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(p.stdout[-2000:], p.stderr[-2000:])
    assert p.returncode == 0 and "K1t ok" in p.stdout
    assert "tc32: smem" in p.stderr   # the tensor-core kernel really ran

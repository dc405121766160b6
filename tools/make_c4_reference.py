"""Run the CPU oracle (oracle/, long double) on BASELINE.json configs[3] (C4: n = 8192,
N(0,1)/sqrt(n), seed 3) and store what the GPU parity test needs: ipiv, the per-step
top-two gaps (rule R3), logabsdet, sign, and 64 seeded sample rows of the inverse.
Calls only oracle/ and synth/.  Output: tests/golden/c4_oracle_ref.npz (~4 MB).
Usage: python tools/make_c4_reference.py [n] [seed] [f32]     (takes ~30-60 min on 8 cores)
With "f32": the oracle on the fp32-rounded input (the f1 path), tol = n u32,
written to tests/golden/f1_oracle_ref_n{n}_s{seed}.npz."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth   # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 3
f32 = len(sys.argv) > 3 and sys.argv[3] == "f32"
A = synth.gen_gaussian(n, seed)
if f32:
    A = A.astype(np.float32)
t0 = time.time()
r = oracle.invert(A, tol=n * (2.0 ** -23 if f32 else 2.0 ** -52))
dt = time.time() - t0
rows = np.sort(np.random.default_rng(12345).choice(n, 64, replace=False))
X = r.inverse[0]
kappa = float(np.abs(A.astype(np.float64)).sum(1).max() * np.abs(X).sum(1).max())
out = os.path.join(ROOT, "tests", "golden", f"{'f1' if f32 else 'c4'}_oracle_ref_n{n}_s{seed}.npz")
np.savez_compressed(out, n=n, seed=seed, ipiv=r.ipiv[0], gap=r.gap[0], logabsdet=r.logabsdet[0], sign=r.sign[0],
                    info=r.info[0], rows=rows, inv_rows=X[rows], kappa_inf=kappa, oracle_seconds=dt,
                    oracle_threads=oracle.threads(),
                    note="written by tools/make_c4_reference.py (oracle/ long-double GJ on [A|I]); synth.gen_gaussian")
print(out, dt, kappa)

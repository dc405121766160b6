"""Time gj_solve (large-n [A | B] path, fp64) against gj_invert at the same n."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for n in [int(x) for x in sys.argv[1:]] or [4096, 8192]:
    A = torch.from_numpy(synth.gen_gaussian(n, seed=3)).cuda()
    X = torch.empty_like(A)
    ti = t(lambda: gj.invert(A, out=X))
    for m in (1, 64, 512):
        B = torch.randn(n, m, dtype=torch.float64, device="cuda")
        ts = t(lambda: gj.solve(A, B))
        fl = 2.0 / 3.0 * n ** 3 + 2.0 * n * n * m
        print(f"n={n} nrhs={m}: solve {ts:.2f} ms ({fl / ts / 1e9:.1f} TFLOP/s nominal)  invert {ti:.2f} ms")

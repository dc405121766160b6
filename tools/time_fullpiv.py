"""Time gj_invert_batched_full (K6) against gj_invert_batched (K1b) on a resident batch."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402


def t(f, reps=5):
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


for dt, n, B in ((torch.float32, 32, 1 << 20), (torch.float64, 32, 1 << 18), (torch.float32, 16, 1 << 20),
                 (torch.float64, 16, 1 << 18), (torch.float32, 8, 1 << 21)):
    A = torch.randn(B, n, n, dtype=dt, device="cuda")
    X = torch.empty_like(A)
    tf = t(lambda: gj.invert_batched_full(A, out=X))
    tp = t(lambda: gj.invert_batched(A, out=X))
    print(f"{dt} n={n} B={B}: full {tf:.3f} ms ({B / tf / 1e3:.3e} mat/s)  partial {tp:.3f} ms  ratio {tf / tp:.2f}")

"""Time gj_solve_batched (K7) on resident batches; GB/s of the algorithmic bytes."""
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


for dt, n, m, B in ((torch.float32, 32, 1, 1 << 20), (torch.float32, 32, 8, 1 << 20), (torch.float32, 32, 32, 1 << 20),
                    (torch.float64, 32, 1, 1 << 18), (torch.float64, 16, 4, 1 << 20)):
    A = torch.randn(B, n, n, dtype=dt, device="cuda")
    R = torch.randn(B, n, m, dtype=dt, device="cuda")
    X = torch.empty_like(R)
    ms = t(lambda: gj.solve_batched(A, R, out=X))
    es = A.element_size()
    gbs = B * (n * n + 2 * n * m) * es / (ms / 1e3) / 1e9
    print(f"{dt} n={n} nrhs={m} B={B}: {ms:.3f} ms  {B / ms * 1e3:.3e} systems/s  {gbs:.0f} GB/s")

# determinant-only run (gj_det on the batched path: K1s without right-hand sides for fp32 n = 32)
for dt, n, B in ((torch.float32, 32, 1 << 20), (torch.float64, 32, 1 << 18)):
    A = torch.randn(B, n, n, dtype=dt, device="cuda")
    ms_det = t(lambda: gj.det(A))
    ms_inv = t(lambda: gj.invert_batched(A))
    print(f"{dt} n={n} B={B}: det-only {ms_det:.3f} ms ({B / ms_det * 1e3:.3e} matrices/s), inverse {ms_inv:.3f} ms")

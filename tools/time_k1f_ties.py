"""Cost of the two-pass K1f run when exact ties are common: C2-sized batches of small-integer
matrices (ties at many steps, so most tasks are redone by the exact pass) and a Gaussian
batch, each timed without ipiv (two passes) and with ipiv (the exact kernel alone).
    python tools/time_k1f_ties.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402

B = 1 << 20
rng = np.random.default_rng(3)
for name, A_host in (("gaussian", rng.standard_normal((B, 32, 32), dtype=np.float32)),
                     ("integers in [-2, 2]", rng.integers(-2, 3, (B, 32, 32)).astype(np.float32)),
                     ("integers in [-50, 50]", rng.integers(-50, 51, (B, 32, 32)).astype(np.float32))):
    A = torch.from_numpy(A_host).cuda()
    X = torch.empty_like(A)
    for ipiv in (False, True):
        run = lambda: gj.invert_batched(A, out=X, ipiv=ipiv, det=False, info=False)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{name:22s} {'exact (ipiv)' if ipiv else 'two-pass':13s}: {np.median(ts):.3f} ms", flush=True)

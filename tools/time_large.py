"""Time gj_invert (large-n blocked path) on N(0,1)/sqrt(n) fp64 matrices: CUDA events on
the launching stream, warm-up first.  Prints GFLOP/s for (2n^3 - n^2) per inversion."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [2048, 4096, 8192]:
    A = torch.from_numpy(synth.gen_gaussian(n, seed=3)).cuda()
    X = torch.empty_like(A)
    gj.invert(A, out=X)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        s.record()
        gj.invert(A, out=X)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = min(ts)
    fl = 2.0 * n ** 3 - n ** 2
    print(f"n={n} ms={t:.2f} GFLOP/s={fl / t / 1e6:.0f}", flush=True)

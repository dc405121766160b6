"""e2e (host buffers) throughput of gj_invert_batched_host on C2 for several chunk sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402

B = 1048576
A = synth.gen_c2(batch=B)
Ah = torch.from_numpy(A).pin_memory()
Xh = torch.empty_like(Ah).pin_memory()
lg = torch.empty(B, dtype=torch.float64).pin_memory()
sg = torch.empty(B, dtype=torch.int8).pin_memory()
for chunk in [int(c) for c in sys.argv[1:]] or [0, 32768, 65536, 131072, 262144]:
    gj.invert_batched_host(Ah, out=Xh, logabsdet=lg, sign=sg, tol=32 * 2.0 ** -23, chunk=chunk)
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        gj.invert_batched_host(Ah, out=Xh, logabsdet=lg, sign=sg, tol=32 * 2.0 ** -23, chunk=chunk)
        ts.append(time.perf_counter() - t0)
    print("  each ms:", [round(x * 1e3, 1) for x in ts])
    t = min(ts)
    print(f"chunk={chunk}: {t * 1e3:.1f} ms  {B / t:.3e} mat/s  {2 * B * 4096 / t / 1e9:.1f} GB/s (H2D+D2H)", flush=True)

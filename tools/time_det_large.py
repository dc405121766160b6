"""gj_det (determinant-only path) vs gj_invert at large n, fp64 and fp32 (CUDA events)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
for dt in (np.float64, np.float32):
    A = torch.from_numpy(synth.gen_gaussian(n, seed=3).astype(dt)).cuda()
    for name, fn in (("invert", lambda: gj.invert(A)), ("det", lambda: gj.det(A))):
        r = fn(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r = fn(); e.record(); torch.cuda.synchronize()
        print(f"{np.dtype(dt).name} n={n} {name}: {s.elapsed_time(e):.2f} ms  logabsdet={float(r.logabsdet):.12f} sign={int(r.sign)}")

"""Time gj_invert on fp32 N(0,1)/sqrt(n) matrices (fp32 panel kernel + tcgen05 TF32 update)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402
for n in [int(a) for a in sys.argv[1:]] or [4096, 8192]:
    A = torch.from_numpy(synth.gen_gaussian(n, seed=3).astype(np.float32)).cuda()
    X = torch.empty_like(A)
    gj.invert(A, out=X)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        s.record(); gj.invert(A, out=X); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    t = min(ts)
    print(f"fp32 n={n} ms={t:.2f} TFLOP/s={(2.0 * n ** 3 - n * n) / t / 1e9:.1f}", flush=True)

"""C3 with K2b vs K2d (GJ_K2_VARIANT is read once per process: run once per variant)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
from tests.parity import compare  # noqa: E402

A, S = synth.gen_c3(return_singular=True)
At = torch.from_numpy(A).cuda()
B = A.shape[0]
X = torch.empty_like(At)
run = lambda: gj.invert_batched(At, tol=synth.C3_TOL, out=X)
r = run()
torch.cuda.synchronize()
info = r.info.cpu().numpy()
print("variant", os.environ.get("GJ_K2_VARIANT"), "flags equal:", np.array_equal(np.nonzero(info)[0], S))
idx = np.arange(0, B, 997)
g = {k: (None if v is None else v[torch.from_numpy(idx).cuda()].cpu().numpy()) for k, v in r._asdict().items()}
ref = oracle.invert_batched(A[idx], tol=synth.C3_TOL)
print(compare(A[idx], g, ref, np.float64, synth.C3_TOL, flat_only=True).summary())
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"C3: {ms:.2f} ms  {B * (2 * 64 ** 3 - 64 ** 2) / (ms / 1e3) / 1e12:.2f} TFLOP/s")

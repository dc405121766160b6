"""Find C2 items whose pivot sequence leaves the oracle's at a step with gap > 1e-6 and
print the step, the oracle's gap, kappa and the GPU's view (diagnostic for the R3 rule)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402
from tests.parity import ipiv_match  # noqa: E402

A = synth.gen_c2()
tol = 32 * 2.0 ** -23
r = gj.invert_batched(torch.from_numpy(A).cuda(), tol=tol)
torch.cuda.synchronize()
ip = r.ipiv.cpu().numpy()
info = r.info.cpu().numpy()
ch = 65536
for c0 in range(0, A.shape[0], ch):
    ref = oracle.invert_batched(A[c0:c0 + ch], tol=tol)
    for b in range(ref.ipiv.shape[0]):
        if ref.info[b] != 0 or info[c0 + b] != 0:
            continue
        ok, ex = ipiv_match(ip[c0 + b], ref.ipiv[b], ref.gap[b])
        if not ok:
            k = int(np.nonzero(ip[c0 + b] != ref.ipiv[b])[0][0])
            Xr = ref.inverse[b]
            kap = np.abs(A[c0 + b].astype(np.float64)).sum(1).max() * np.abs(Xr).sum(1).max()
            print(f"item {c0 + b}: first mismatch step {k}: gpu q={ip[c0 + b][k]} oracle q={ref.ipiv[b][k]} "
                  f"oracle gap {ref.gap[b][k]:.3e} (gaps around: {np.array2string(ref.gap[b][max(0, k - 2):k + 3], precision=2)}) "
                  f"kappa_inf {kap:.3e} kappa*eps32 {kap * 2.0 ** -23:.3e}")

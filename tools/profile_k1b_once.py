"""C2-shaped K1b launches for an ncu capture (Gaussian fp32 32x32, 1,048,576 items, drawn on
the device — the capture needs the kernel's behaviour, not the C2 bytes).  Called like the
bench (no ipiv), so this runs K1f (gj_blk32_kernel<2,4,2,1>) plus the exact pass over the
(empty) tie list; `exact` as argument requests ipiv and runs the exact kernel (<2,4,2,0>)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402

exact = len(sys.argv) > 1 and sys.argv[1] == "exact"
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((1 << 20, 32, 32), generator=g, device="cuda", dtype=torch.float32)
X = torch.empty_like(A)
for _ in range(3):
    gj.invert_batched(A, out=X, ipiv=exact, det=False, info=False)
torch.cuda.synchronize()
print("ok")

"""C2-shaped K1b launches for an ncu capture (Gaussian fp32 32x32, 1,048,576 items, drawn on
the device — the capture needs the kernel's behaviour, not the C2 bytes)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((1 << 20, 32, 32), generator=g, device="cuda", dtype=torch.float32)
X = torch.empty_like(A)
for _ in range(3):
    gj.invert_batched(A, out=X)
torch.cuda.synchronize()
print("ok")

import sys
import torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
A = torch.randn(1 << 16, 64, 64, dtype=torch.float64, device="cuda")
X = torch.empty_like(A)
gj.invert_batched(A, out=X)
torch.cuda.synchronize()

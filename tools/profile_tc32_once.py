import os, sys
os.environ["GJ_K1_TC"] = "1"
import torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
A = torch.randn(1 << 18, 32, 32, device="cuda")
X = torch.empty_like(A)
gj.invert_batched(A, out=X)
torch.cuda.synchronize()

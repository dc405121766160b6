"""One C2-sized launch each of gj_invert_batched_full (K6) and gj_solve_batched (K7) for
ncu (tools/run_ncu_f2_f4.sh)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402

A = torch.randn(1 << 20, 32, 32, device="cuda")
X = torch.empty_like(A)
B = torch.randn(1 << 20, 32, 1, device="cuda")
gj.invert_batched_full(A, out=X)
gj.solve_batched(A, B)
torch.cuda.synchronize()

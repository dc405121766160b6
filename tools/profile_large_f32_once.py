"""One fp32 gj_invert of an n x n N(0,1)/sqrt(n) matrix (for ncu launch lists)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.from_numpy(synth.gen_gaussian(n, seed=3).astype(np.float32)).cuda()
X = torch.empty_like(A)
gj.invert(A, out=X)
torch.cuda.synchronize()
print("done", n)

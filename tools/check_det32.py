import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.from_numpy(synth.gen_gaussian(n, seed=3).astype(np.float32)).cuda()
outs = []
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    r = gj.invert(A)
    torch.cuda.synchronize()
    outs.append((float(r.logabsdet), r.ipiv.cpu().numpy(), r.inverse.cpu().numpy()))
    print(i, outs[-1][0], flush=True)
for i in range(1, len(outs)):
    d = np.nonzero(outs[0][1] != outs[i][1])[0]
    print("ipiv equal", len(d) == 0, "first diff", d[:1], "inverse equal", np.array_equal(outs[0][2], outs[i][2]))
d = gj.det(A); torch.cuda.synchronize(); print("det", float(d.logabsdet))

import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1401_7962_b200 as gj, oracle, synth
from tests.parity import compare
A = synth.gen_normal_batch(1037, 32, seed=5, dtype=np.float32)
r = gj.invert_batched(torch.from_numpy(A).cuda(), tol=32 * 2.0 ** -23)
torch.cuda.synchronize()
g = {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}
ref = oracle.invert_batched(A, tol=32 * 2.0 ** -23)
rep = compare(A, g, ref, np.float32, 32 * 2.0 ** -23)
print(rep.summary())

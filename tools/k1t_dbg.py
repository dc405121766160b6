import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1401_7962_b200 as gj, oracle, synth
rng = np.random.default_rng(3)
B = synth.gen_normal_batch(1000, 32, seed=22, dtype=np.float32)
S = rng.choice(1000, 60, replace=False)
for b in S: B[b, 7] = B[b, 3]
B[S[0]] = 0.0
r = gj.invert_batched(torch.from_numpy(B).cuda(), tol=1e-5); torch.cuda.synchronize()
info = r.info.cpu().numpy(); ref = oracle.invert_batched(B, tol=1e-5)
bad = np.nonzero((info != 0) != (ref.info != 0))[0]
print("bad", bad, info[bad], ref.info[bad], "S0", S[0], info[S[0]], ref.info[S[0]])
for b in bad:
    print(b, "in S" if b in S else "regular", "cmin", np.nanmin(ref.cmax_rel[b]))
    lg = r.logabsdet.cpu().numpy()[b]; print("lg", lg, ref.logabsdet[b])

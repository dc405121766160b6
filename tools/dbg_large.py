import numpy as np, torch, sys
sys.path.insert(0, '.')
import synth, paper_1401_7962_b200 as gj
for n in [int(a) for a in sys.argv[1:]]:
    A = torch.from_numpy(synth.gen_gaussian(n, seed=40 + n)).cuda()
    r = gj.invert(A)
    torch.cuda.synchronize()
    print(n, "ok", float(r.logabsdet), flush=True)

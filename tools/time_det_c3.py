"""C3-sized fp64 n = 64 batch: det-only (gj_det, K2f without the D columns) vs the inverse; bitwise equality of the det outputs and both times."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj, synth
A = torch.from_numpy(synth.gen_c3()).cuda()
r1 = gj.invert_batched(A, tol=synth.C3_TOL); r2 = gj.det(A, tol=synth.C3_TOL); torch.cuda.synchronize()
for k in ("logabsdet", "sign", "det", "ipiv", "info"):
    print(k, torch.equal(getattr(r1, k), getattr(r2, k)))
def t(f):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[3]
print("inverse", t(lambda: gj.invert_batched(A, tol=synth.C3_TOL)), "det-only", t(lambda: gj.det(A, tol=synth.C3_TOL)))

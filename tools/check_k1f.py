"""K1f (the two-pass fp32 n = 32 run without ipiv) against the exact kernel (the same call
with ipiv): every output bitwise equal, on batches with and without exact ties, singular
items, an odd batch and an inverse that aliases A.   python tools/check_k1f.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402


def batch(kind, B, seed):
    rng = np.random.default_rng(seed)
    if kind == "gauss":
        A = rng.standard_normal((B, 32, 32)).astype(np.float32)
    elif kind == "int":      # small integers: exact ties in many steps
        A = rng.integers(-3, 4, (B, 32, 32)).astype(np.float32)
    elif kind == "mixed":    # a few tie / singular items among Gaussian ones
        A = rng.standard_normal((B, 32, 32)).astype(np.float32)
        idx = rng.choice(B, B // 50, replace=False)
        A[idx] = rng.integers(-2, 3, (len(idx), 32, 32)).astype(np.float32)
        A[idx[:5], :, 7] = 0.0                       # zero column: singular
        H = np.stack([synth.hadamard_pd(32, seed=s)[0] for s in range(3)]).astype(np.float32)
        A[idx[5:8]] = H
    return A


def run(A, ipiv, alias=False):
    X = A.clone() if alias else torch.empty_like(A)
    src = X if alias else A
    r = gj.invert_batched(src, out=X, ipiv=ipiv)
    torch.cuda.synchronize()
    return [t.cpu() for t in (r.inverse, r.logabsdet, r.sign, r.det, r.info)]


ok = True
for kind, B in (("gauss", 100001), ("int", 4097), ("mixed", 65537)):
    A = torch.from_numpy(batch(kind, B, 11)).cuda()
    ref = run(A, True)
    for alias in (False, True):
        got = run(A, False, alias)
        same = all(torch.equal(a.view(torch.int32) if a.dtype == torch.float32 else a,
                               b.view(torch.int32) if b.dtype == torch.float32 else b) for a, b in zip(ref, got))
        print(f"{kind:6s} B={B} alias={alias}: bitwise equal to the exact kernel: {same}", flush=True)
        ok &= same
print("K1F CHECK", "PASS" if ok else "FAIL")

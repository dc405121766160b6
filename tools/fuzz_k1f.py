"""Randomised sweep of the two-pass fp32 n = 32 runs (K1f inverse, K1s solve / det): for random
batch sizes, value families and tie densities, every output of the call WITHOUT ipiv must be
bitwise that of the same call with ipiv (the exact kernels).  python tools/fuzz_k1f.py [trials]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(1234)
fails = 0
kinds = ["gauss", "int2", "int5", "scaled", "lowrank", "dup", "mixed", "uniform01"]


def make(kind, B):
    if kind == "gauss":
        return rng.standard_normal((B, 32, 32))
    if kind == "int2":
        return rng.integers(-2, 3, (B, 32, 32)).astype(np.float64)
    if kind == "int5":
        return rng.integers(-5, 6, (B, 32, 32)).astype(np.float64)
    if kind == "scaled":
        return rng.standard_normal((B, 32, 32)) * 10.0 ** rng.uniform(-20, 20, (B, 1, 32))
    if kind == "lowrank":
        U = rng.standard_normal((B, 32, 31))
        return U @ rng.standard_normal((B, 31, 32))
    if kind == "dup":
        A = rng.standard_normal((B, 32, 32))
        A[:, 5] = A[:, 9]
        return A
    if kind == "uniform01":
        return rng.uniform(0, 1, (B, 32, 32))
    A = rng.standard_normal((B, 32, 32))
    idx = rng.choice(B, max(1, B // 10), replace=False)
    A[idx] = rng.integers(-1, 2, (len(idx), 32, 32))
    return A


def bits(t):
    return t.view(torch.int32) if t.dtype == torch.float32 else t


for t in range(trials):
    kind = kinds[t % len(kinds)]
    B = int(rng.choice([1, 2, 3, 7, 63, 64, 65, 1000, 4097, int(rng.integers(1, 70000))]))
    A = torch.from_numpy(make(kind, B).astype(np.float32)).cuda()
    tol = float(rng.choice([0.0, 1e-7, 32 * 2.0 ** -23, 1e-3]))
    r = gj.invert_batched(A, tol=tol)
    f = gj.invert_batched(A, tol=tol, ipiv=False)
    d0, d1 = gj.det(A, tol=tol), gj.det(A, tol=tol, ipiv=False)
    Bm = torch.from_numpy(rng.standard_normal((B, 32, 2)).astype(np.float32)).cuda()
    s0, s1 = gj.solve_batched(A, Bm, tol=tol), gj.solve_batched(A, Bm, tol=tol, ipiv=False)
    torch.cuda.synchronize()
    ok = all(torch.equal(bits(getattr(r, k)), bits(getattr(f, k))) for k in ("inverse", "logabsdet", "sign", "det", "info"))
    ok &= all(torch.equal(bits(getattr(d0, k)), bits(getattr(d1, k))) for k in ("logabsdet", "sign", "det", "info"))
    ok &= all(torch.equal(bits(getattr(s0, k)), bits(getattr(s1, k))) for k in ("X", "logabsdet", "sign", "info"))
    if not ok:
        fails += 1
        print(f"trial {t}: kind={kind} B={B} tol={tol}: MISMATCH", flush=True)
print(f"{trials} trials, {fails} mismatching")

"""One small launch of every kernel family, each checked against torch.linalg on the device —
the quick all-families check (compute-sanitizer is closed on this pool):
    python tools/families_smoke.py [family ...]
Families: k1b k1 k2 k2f k1s k6 k7 large large32 det host."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator(device="cuda").manual_seed(7)


def rnd(*shape, dtype=torch.float64):
    return torch.randn(*shape, generator=g, device=dev, dtype=torch.float64).to(dtype)


def check(name, X, A, tol):
    ref = torch.linalg.inv(A.double())
    err = ((X.double() - ref).abs().amax() / ref.abs().amax()).item()
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err < tol, name


fams = sys.argv[1:] or ["k1b", "k1", "k2", "k2f", "k1s", "k6", "k7", "large", "large32", "det", "host"]
for f in fams:
    if f == "k1b":      # fp32 n = 32: two rows per lane, TMA, blocked (odd batch: a half-empty warp task)
        A = rnd(37, 32, 32, dtype=torch.float32)
        check(f, gj.invert_batched(A).inverse, A, 2e-3)
    elif f == "k1":     # fp64 n = 16 and fp32 n = 20 (padded rows)
        A = rnd(33, 16, 16)
        check(f + "/f64n16", gj.invert_batched(A).inverse, A, 1e-10)
        A = rnd(9, 20, 20, dtype=torch.float32)
        check(f + "/f32n20", gj.invert_batched(A).inverse, A, 2e-3)
    elif f == "k2":     # 33..64
        A = rnd(11, 48, 48)
        check(f, gj.invert_batched(A).inverse, A, 1e-10)
    elif f == "k2f":    # fp64 n = 64: panel warp + DMMA warp, shared-memory resident
        A = rnd(13, 64, 64)
        check(f, gj.invert_batched(A).inverse, A, 1e-10)
    elif f == "k1s":    # fp32 n = 32 solve
        A = rnd(19, 32, 32, dtype=torch.float32)
        B = rnd(19, 32, 3, dtype=torch.float32)
        Xs = gj.solve_batched(A, B).X
        ref = torch.linalg.solve(A.double(), B.double())
        print(f"{f}: rel err {((Xs.double() - ref).abs().amax() / ref.abs().amax()).item():.2e}", flush=True)
    elif f == "k6":     # full pivoting
        A = rnd(21, 32, 32, dtype=torch.float32)
        check(f, gj.invert_batched_full(A).inverse, A, 2e-3)
    elif f == "k7":     # multi-RHS solve, fp64
        A = rnd(7, 24, 24)
        B = rnd(7, 24, 5)
        Xs = gj.solve_batched(A, B).X
        ref = torch.linalg.solve(A, B)
        print(f"{f}: rel err {((Xs - ref).abs().amax() / ref.abs().amax()).item():.2e}", flush=True)
    elif f == "large":  # leaf cluster kernel + K4b DMMA GEMM + un-permutation (ragged n)
        A = rnd(300, 300)
        check(f, gj.invert(A).inverse, A, 1e-10)
    elif f == "large32":  # fp32 on tcgen05
        A = rnd(384, 384, dtype=torch.float32)
        check(f, gj.invert(A).inverse, A, 5e-3)
    elif f == "det":
        A = rnd(300, 300)
        r = gj.det(A)
        ref = torch.linalg.slogdet(A)
        print(f"{f}: logabsdet diff {abs(float(r.logabsdet) - ref.logabsdet.item()):.2e}", flush=True)
    elif f == "host":   # host-buffer pipeline
        A = rnd(70, 32, 32, dtype=torch.float32).cpu()
        X = torch.empty_like(A)
        gj.invert_batched_host(A, out=X)
        check(f, X.to(dev), A.to(dev), 2e-3)
torch.cuda.synchronize()
print("sanitize workload done")

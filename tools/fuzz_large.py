"""Randomised parity sweep of the single-matrix (large-n) path against the oracle
(`python tools/fuzz_large.py TRIALS SEED`): random order n in 65..1400 (ragged against the
32-row leaf and the 128-column panel), dtype, family (Gaussian / sqrt(n), graded rows,
small integers with ties, diagonally dominant), through gj_invert, gj_det and gj_solve
(1..40 right-hand sides); R1 (kappa rule), R3 (pivot sequence with G26's threshold), R4,
R5 and the solve residual against the oracle's solution."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_7962_b200 as gj  # noqa: E402
from tests.parity import ipiv_match, tie_gap  # noqa: E402

EPS = {np.float32: 2.0 ** -23, np.float64: 2.0 ** -52}


def main(trials, seed):
    rng = np.random.default_rng(seed)
    fails = 0
    for tr in range(trials):
        dtype = [np.float32, np.float64][rng.integers(2)]
        n = int(rng.integers(65, 1401))
        kind = ["gauss", "graded", "int", "diagdom"][rng.integers(4)]
        A = rng.standard_normal((n, n)) / np.sqrt(n)
        if kind == "graded":
            A *= 10.0 ** rng.uniform(-3, 3, (n, 1))
        elif kind == "int":
            A = rng.integers(-3, 4, (n, n)).astype(np.float64)
        elif kind == "diagdom":
            A += 2 * np.eye(n)
        A = A.astype(dtype)
        m = int(rng.integers(1, 41))
        Bm = rng.standard_normal((n, m)).astype(dtype)
        At = torch.from_numpy(A).cuda()
        tol = n * EPS[dtype]   # the library default, passed to both sides
        r = gj.invert(At, tol=tol)
        d = gj.det(At, tol=tol)
        s = gj.solve(At, torch.from_numpy(Bm).cuda(), tol=tol)
        torch.cuda.synchronize()
        ref = oracle.invert(A, tol=tol)
        msgs = []
        tag = f"trial {tr}: {dtype.__name__} n={n} {kind} m={m}"
        if ref.info[0] != 0 or int(r.info.item()) != 0:
            cmin = np.nanmin(np.where(np.isnan(ref.cmax_rel[0]), np.inf, ref.cmax_rel[0]))
            if (ref.info[0] != 0) != (int(r.info.item()) != 0) and not (tol / 10 <= cmin <= 10 * tol):
                msgs.append(f"flag gpu {int(r.info.item())} oracle {ref.info[0]} cmin {cmin:.2e}")
        else:
            Xr = ref.inverse[0]
            kap = np.abs(A.astype(np.float64)).sum(1).max() * np.abs(Xr).sum(1).max()
            e = np.abs(r.inverse.cpu().numpy().astype(np.float64) - Xr).max() / np.abs(Xr).max()
            if kap * EPS[dtype] < 0.1 and e > max(2e-4 if dtype == np.float32 else 1e-10, kap * EPS[dtype]):
                msgs.append(f"inverse e {e:.2e} kappa eps {kap * EPS[dtype]:.2e}")
            if not ipiv_match(r.ipiv.cpu().numpy(), ref.ipiv[0], ref.gap[0], thr=tie_gap(dtype, n))[0]:
                msgs.append("ipiv")
            if int(r.sign.item()) != int(ref.sign[0]) and kap * EPS[dtype] < 0.1:
                msgs.append("sign")
            if abs(float(r.logabsdet.item()) - ref.logabsdet[0]) > max(1e-10, kap * EPS[dtype]):
                msgs.append("logabsdet")
            for k in ("logabsdet", "sign", "ipiv", "info"):
                if not torch.equal(getattr(r, k), getattr(d, k)):
                    msgs.append(f"det-only {k}")
            Xs = s.X.cpu().numpy().astype(np.float64)
            Xo = Xr @ Bm.astype(np.float64)
            es = np.abs(Xs - Xo).max() / np.abs(Xo).max()
            if kap * EPS[dtype] < 0.1 and es > 4 * max(2e-4 if dtype == np.float32 else 1e-10, kap * EPS[dtype]):
                msgs.append(f"solve e {es:.2e}")
        if msgs:
            fails += 1
            print(tag, "|", "; ".join(msgs), flush=True)
    print(f"fuzz large: {trials} trials, {fails} failing", flush=True)
    return fails


if __name__ == "__main__":
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    sd = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    sys.exit(1 if main(t, sd) else 0)

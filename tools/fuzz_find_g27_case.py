"""Replay the randomised sweep's input stream (tools/fuzz_batched.py, same RNG consumption)
for the given seeds and pull out fp32 n = 64 small-integer items whose GPU pivot sequence
leaves the oracle's at an oracle gap ABOVE reading G26's n u but below G27's 100 n u (the
divergence found by seeds 7/8 in round 1, profiles/r01_fuzz.md).  Writes the first such
item to tests/golden/g27_fp32_n64_case.npz (the matrix and its provenance only — the test
recomputes both sides).  Runs on the GPU box:  python tools/fuzz_find_g27_case.py 7 8"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle  # noqa: E402
import paper_1401_7962_b200 as gj  # noqa: E402
from fuzz_batched import EPS, family  # noqa: E402
from tests.parity import tie_gap  # noqa: E402

KINDS = ["gauss", "graded", "int", "nearsing", "singular", "diagdom", "perm"]


def replay(seed, trials=400):
    rng = np.random.default_rng(seed)
    for tr in range(trials):
        dtype = [np.float32, np.float64][rng.integers(2)]
        n = int(rng.choice([1, 2, 3, 5, 8, 13, 16, 17, 24, 31, 32, 33, 40, 47, 63, 64]))
        B = int(rng.integers(1, 1500))
        kind = KINDS[rng.integers(len(KINDS))]
        tol = float(n * EPS[dtype]) if rng.integers(2) else float(10.0 ** rng.uniform(-12, -4))
        A = family(rng, kind, B, n, dtype)
        if n <= 32:
            m = int(rng.integers(1, 33)) if rng.integers(2) else int(rng.integers(1, 9))
            rng.standard_normal((B, n, m))
        yield tr, dtype, n, B, kind, tol, A


def main(seeds):
    out = os.environ.get("G27_OUT", os.path.join(ROOT, "tests", "golden", "g27_fp32_n64_case.npz"))
    for seed in seeds:
        for tr, dtype, n, B, kind, tol, A in replay(seed):
            if not (dtype == np.float32 and n == 64 and kind == "int"):
                continue
            r = gj.invert_batched(torch.from_numpy(A).cuda(), tol=tol)
            torch.cuda.synchronize()
            ip = r.ipiv.cpu().numpy()
            ref = oracle.invert_batched(A, tol=tol)
            lo, hi = tie_gap(dtype, n), 100 * n * EPS[dtype] / 2
            for b in range(B):
                if ref.info[b] != 0:
                    continue
                neq = np.nonzero(ip[b] != ref.ipiv[b])[0]
                if len(neq) and lo < ref.gap[b][neq[0]] < hi:
                    k = int(neq[0])
                    print(f"seed {seed} trial {tr} item {b}: first divergence at step {k + 1}, "
                          f"oracle gap {ref.gap[b][k]:.3e} (G26 {lo:.2e}, G27 {hi:.2e})", flush=True)
                    np.savez_compressed(out, A=A[b], tol=tol, seed=seed, trial=tr, item=b, step=k,
                                        note="tools/fuzz_find_g27_case.py: input of tools/fuzz_batched.py seed/trial/"
                                             "item (family 'int': integers in [-3, 3], fp32, n = 64)")
                    return 0
    print("no case found", flush=True)
    return 1


if __name__ == "__main__":
    sys.exit(main([int(s) for s in sys.argv[1:]] or [7, 8]))

"""Randomised parity sweep of the batched entry points against the oracle (evidence run,
not a test: `python tools/fuzz_batched.py [trials] [seed]`).  Per trial: a dtype, an order
n in 1..64, a batch size (ragged against every kernel's task size) and an input family —
Gaussian, graded rows (1e-6..1e6), small integers (exact ties), near-singular (a row
duplicated and perturbed by 1e-9), exactly singular items mixed in, diagonally dominant,
scaled signed permutations, all-zero items — through gj_invert_batched (K1/K1b/K2/K2f),
gj_det, gj_solve_batched (K1s/K7, n <= 32) and full pivoting (K6, n <= 32), compared with
the oracle under the rules of tests/parity.py.  Prints one line per failing trial and a
summary."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_7962_b200 as gj  # noqa: E402
from tests.parity import compare, ipiv_match, tie_gap  # noqa: E402

VERBOSE = False
EXEMPT = {}   # pivot divergences exempted by G27, by rule (reported next to the strict result)
EPS = {np.float32: 2.0 ** -23, np.float64: 2.0 ** -52}


def family(rng, kind, B, n, dtype):
    A = rng.standard_normal((B, n, n))
    if kind == "graded":
        A *= 10.0 ** rng.uniform(-6, 6, (B, n, 1))
    elif kind == "int":
        A = rng.integers(-3, 4, (B, n, n)).astype(np.float64)
    elif kind == "nearsing" and n > 1:
        i, j = rng.choice(n, 2, replace=False)
        A[:, j] = A[:, i] + 1e-9 * rng.standard_normal((B, n))
    elif kind == "singular" and n > 1:
        S = rng.choice(B, max(1, B // 10), replace=False)
        A[S, 0] = A[S, n - 1]
        A[S[0]] = 0.0
    elif kind == "diagdom":
        A += 2 * n * np.eye(n)
    elif kind == "perm":
        A = np.zeros((B, n, n))
        for b in range(B):
            A[b, np.arange(n), rng.permutation(n)] = rng.choice([-4.0, -0.5, 0.25, 2.0], n)
    return A.astype(dtype)


def main(trials=120, seed=0):
    rng = np.random.default_rng(seed)
    kinds = ["gauss", "graded", "int", "nearsing", "singular", "diagdom", "perm"]
    fails = 0
    for tr in range(trials):
        dtype = [np.float32, np.float64][rng.integers(2)]
        n = int(rng.choice([1, 2, 3, 5, 8, 13, 16, 17, 24, 31, 32, 33, 40, 47, 63, 64]))
        B = int(rng.integers(1, 1500))
        kind = kinds[rng.integers(len(kinds))]
        tol = float(n * EPS[dtype]) if rng.integers(2) else float(10.0 ** rng.uniform(-12, -4))
        A = family(rng, kind, B, n, dtype)
        At = torch.from_numpy(A).cuda()
        tag = f"trial {tr}: {dtype.__name__} n={n} B={B} {kind} tol={tol:.1e}"
        if VERBOSE:
            print("start", tag, flush=True)
        msgs = []
        # inverse
        r = gj.invert_batched(At, tol=tol)
        d = gj.det(At, tol=tol)
        torch.cuda.synchronize()
        g = {k: (None if v is None else v.cpu().numpy()) for k, v in r._asdict().items()}
        ref = oracle.invert_batched(A, tol=tol)
        rep = compare(A, g, ref, dtype, tol)
        # reading G27: singular-flag decisions below the kernel precision's resolution (the
        # oracle's smallest relative pivot and the threshold both under 100 n u(dtype): the
        # rounding noise of a computed pivot, growth included) are not determined; items that
        # are numerically singular in the dtype (kappa eps >= 0.1, R4's exemption) have no
        # meaningful inverse to compare
        res = 100 * n * EPS[dtype] / 2
        cmin = np.nanmin(np.where(np.isnan(ref.cmax_rel), np.inf, ref.cmax_rel), axis=1)
        unres = (cmin < res) & (tol < res)
        kap0 = np.full(B, np.inf)
        ok0 = ref.info == 0
        kap0[ok0] = np.abs(A[ok0].astype(np.float64)).sum(2).max(1) * np.abs(ref.inverse[ok0]).sum(2).max(1)
        unres |= kap0 * EPS[dtype] >= 0.1   # numerically singular in the dtype: flag not determined
        rep.info_fail = [b for b in rep.info_fail if not unres[b]]
        if VERBOSE and rep.info_fail:
            for b in rep.info_fail[:3]:
                print(f"   info item {b}: gpu {g['info'][b]} oracle {ref.info[b]} oracle cmin {cmin[b]:.3e} "
                      f"oracle min step {np.nanargmin(ref.cmax_rel[b])} tol {tol:.2e}", flush=True)
        kap = np.full(B, np.inf)
        okr = ref.info == 0
        kap[okr] = np.abs(A[okr].astype(np.float64)).sum(2).max(1) * np.abs(ref.inverse[okr]).sum(2).max(1)
        numsing = kap * EPS[dtype] >= 0.1
        rep.inv_kappa_fail = [b for b in rep.inv_kappa_fail if not numsing[b]]
        # G27 for pivots: a divergence at an oracle gap under 100 n u (the rounding
        # noise with growth) is not determined at the kernel's precision, and neither is any step
        # after the first one whose oracle pivot is below that resolution (its candidates are
        # rounding noise); counted separately from the strict R3 / G26 result
        def first_unresolved(b, rf=ref):
            low = np.nonzero(np.nan_to_num(rf.cmax_rel[b], nan=np.inf) < res)[0]
            return int(low[0]) if len(low) else n

        def undetermined(b, gip=g["ipiv"], rf=ref):
            k0 = first_unresolved(b)
            if k0 < n:
                ok, _ = ipiv_match(gip[b][:k0], rf.ipiv[b][:k0], rf.gap[b][:k0], thr=tie_gap(dtype, n))
                if ok:
                    return "after_unresolved_pivot"
            if ipiv_match(gip[b], rf.ipiv[b], rf.gap[b], thr=max(tie_gap(dtype, n), res))[0]:
                return "gap_under_100nu"
            return None
        strict_fail = len(rep.ipiv_fail)
        kinds_ex = [undetermined(b) for b in rep.ipiv_fail]
        rep.ipiv_fail = [b for b, kx in zip(rep.ipiv_fail, kinds_ex) if kx is None]
        for kx in kinds_ex:
            if kx is not None:
                EXEMPT[kx] = EXEMPT.get(kx, 0) + 1
        EXEMPT["strict_r3_g26_fail"] = EXEMPT.get("strict_r3_g26_fail", 0) + strict_fail
        if rep.info_fail or rep.ipiv_fail or rep.sign_fail or rep.logdet_fail or rep.inv_kappa_fail:
            msgs.append("invert: " + rep.summary())
        for k in ("logabsdet", "sign", "ipiv", "info"):
            if not torch.equal(getattr(r, k), getattr(d, k)):
                msgs.append(f"det-only {k} differs from the inverting path")
        if n <= 32:
            m = int(rng.integers(1, 33)) if rng.integers(2) else int(rng.integers(1, 9))
            Bm = rng.standard_normal((B, n, m)).astype(dtype)
            s = gj.solve_batched(At, torch.from_numpy(Bm).cuda(), tol=tol)
            f = gj.invert_batched_full(At, tol=tol)
            torch.cuda.synchronize()
            rs = oracle.solve_batched(A, Bm, tol=tol)
            ok = (rs.info == 0) & (s.info.cpu().numpy() == 0)
            if not np.array_equal(s.info.cpu().numpy() != 0, rs.info != 0):
                cmin = np.nanmin(np.where(np.isnan(ref.cmax_rel), np.inf, ref.cmax_rel), axis=1)
                band = (cmin >= tol / 10) & (cmin <= tol * 10)
                if np.any(((s.info.cpu().numpy() != 0) != (rs.info != 0)) & ~band & ~unres):
                    msgs.append("solve: singular flags differ")
            if ok.any():
                Ai = ref.inverse[ok]
                kap = np.abs(A[ok].astype(np.float64)).sum(2).max(1) * np.abs(Ai).sum(2).max(1)
                X = s.X.cpu().numpy()[ok].astype(np.float64)
                e = np.abs(X - rs.X[ok]).max(axis=(1, 2)) / np.maximum(np.abs(rs.X[ok]).max(axis=(1, 2)), 1e-300)
                lim = np.maximum(2e-4 if dtype == np.float32 else 1e-10, kap * EPS[dtype])
                lim[kap * EPS[dtype] >= 0.1] = np.inf
                if np.any(e > lim):
                    msgs.append(f"solve m={m}: max e/lim {np.max(e / lim):.2f}")
                sip = s.ipiv.cpu().numpy()
                bad = [b for b in np.nonzero(ok)[0]
                       if not ipiv_match(sip[b], rs.ipiv[b], rs.gap[b], thr=max(tie_gap(dtype, n), res))[0]
                       and kap0[b] * EPS[dtype] < 0.1]
                if bad:
                    msgs.append(f"solve ipiv: {len(bad)} items")
            gf = {k: (None if v is None else v.cpu().numpy()) for k, v in f._asdict().items()}
            reff = oracle.invert_full_batched(A, tol=tol)
            repf = compare(A, gf, reff, dtype, tol)
            cminf = np.nanmin(np.where(np.isnan(reff.cmax_rel), np.inf, reff.cmax_rel), axis=1)
            repf.info_fail = [b for b in repf.info_fail if not ((cminf[b] < res) and (tol < res))]
            repf.inv_kappa_fail = [b for b in repf.inv_kappa_fail if not numsing[b]]
            if repf.info_fail or repf.ipiv_fail or repf.sign_fail or repf.logdet_fail or repf.inv_kappa_fail:
                msgs.append("full: " + repf.summary())
        if msgs:
            fails += 1
            print(tag, "|", " ; ".join(msgs), flush=True)
    print(f"fuzz: {trials} trials, {fails} failing; pivot divergences beyond R3/G26 and their G27 "
          f"classification: {EXEMPT}", flush=True)
    return fails


if __name__ == "__main__":
    import os
    VERBOSE = bool(os.environ.get("FUZZ_VERBOSE"))
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    sd = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    sys.exit(1 if main(t, sd) else 0)

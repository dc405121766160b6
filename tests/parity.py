"""Parity rules R1–R8 comparing GPU outputs with the oracle.

Test-side helper: imports the oracle's result type only through duck typing, never the
product package."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

EPS = {np.float32: 2.0 ** -23, np.float64: 2.0 ** -52}
TOL_INV = {np.float32: 2e-4, np.float64: 1e-10}      # BASELINE.json north_star
TOL_RES = {np.float32: 1e-3, np.float64: 1e-9}       # BASELINE.json north_star
TIE_GAP = 1e-6                                        # north_star "top two ... differ by > 1e-6 relative"


def tie_gap(dtype, n: int) -> float:
    """R3 exemption threshold (reading G26): the north star's 1e-6, raised to
    gamma_n = n u (u = unit roundoff of the kernel's dtype) — the standard bound on the
    rounding error of a computed Schur-complement entry relative to its column — so that a
    decision the kernel's own precision cannot resolve is not required to match the exact
    one.  fp64: gamma_32 = 7e-15, the 1e-6 governs; fp32 n = 32: 1.9e-6."""
    u = {np.float32: 2.0 ** -24, np.float64: 2.0 ** -53}[np.dtype(dtype).type]
    return max(TIE_GAP, n * u)


@dataclass
class Report:
    n_items: int = 0
    n_singular_ref: int = 0
    inv_flat_fail: list = field(default_factory=list)
    inv_kappa_fail: list = field(default_factory=list)
    ipiv_fail: list = field(default_factory=list)
    ipiv_tie_exempt: int = 0          # items whose pivots leave the oracle's at a gap <= 1e-6 (G12)
    ipiv_g26_exempt: int = 0          # ... at a gap in (1e-6, n u] (reading G26's raised band)
    ipiv_g26_items: list = field(default_factory=list)
    sign_fail: list = field(default_factory=list)
    logdet_fail: list = field(default_factory=list)
    det_fail: list = field(default_factory=list)
    info_fail: list = field(default_factory=list)
    max_inv_err: float = 0.0
    max_inv_err_over_keps: float = 0.0
    max_logdet_err: float = 0.0

    def summary(self) -> str:
        return (f"items={self.n_items} singular_ref={self.n_singular_ref} inv_flat_fail={len(self.inv_flat_fail)} "
                f"inv_kappa_fail={len(self.inv_kappa_fail)} ipiv_fail={len(self.ipiv_fail)} "
                f"ipiv_tie_exempt={self.ipiv_tie_exempt} ipiv_g26_exempt={self.ipiv_g26_exempt} sign_fail={len(self.sign_fail)} "
                f"logdet_fail={len(self.logdet_fail)} det_fail={len(self.det_fail)} info_fail={len(self.info_fail)} "
                f"max_inv_err={self.max_inv_err:.3e} max_e/(k*eps)={self.max_inv_err_over_keps:.3e} "
                f"max_dlogdet={self.max_logdet_err:.3e}")


def ipiv_match(ipiv_gpu, ipiv_ref, gap_ref, jpiv_gpu=None, jpiv_ref=None, thr=TIE_GAP):
    """R3: equal step by step; at the first mismatch the oracle's gap_k must be <= thr
    (1e-6, or tie_gap(dtype, n)) and later steps are not compared.  Full pivoting: a step matches when both its row
    and its column swap match.  Returns (ok, exempted)."""
    diff = ipiv_gpu != ipiv_ref
    if jpiv_gpu is not None:
        diff = diff | (jpiv_gpu != jpiv_ref)
    neq = np.nonzero(diff)[0]
    if len(neq) == 0:
        return True, False
    k = neq[0]
    return bool(gap_ref[k] <= thr), True


def first_divergence_gap(ipiv_gpu, ipiv_ref, gap_ref):
    """The oracle's top-two gap at the first step where the pivots differ (None if equal)."""
    neq = np.nonzero(ipiv_gpu != ipiv_ref)[0]
    return None if len(neq) == 0 else float(gap_ref[neq[0]])


def compare(A, gpu, ref, dtype, tol, kappa=None, check_ipiv=True, check_det=False, det_rtol=1e-12,
            flat_only=False) -> Report:
    """A: [B,n,n] inputs; gpu: dict of numpy arrays (inverse, ipiv, logabsdet, sign, det, info);
    ref: oracle result.  ``flat_only``: every regular item must meet the flat R1 bound."""
    dtype = np.dtype(dtype).type
    eps = EPS[dtype]
    B = A.shape[0]
    rep = Report(n_items=B)
    ref_sing = ref.info != 0
    rep.n_singular_ref = int(ref_sing.sum())
    # R7: singular flag, with the [tol/10, 10 tol] band exemption
    gpu_sing = gpu["info"] != 0
    with np.errstate(invalid="ignore"):
        cmin = np.nanmin(np.where(np.isnan(ref.cmax_rel), np.inf, ref.cmax_rel), axis=1)
    band = (cmin >= tol / 10) & (cmin <= tol * 10)
    bad = np.nonzero((gpu_sing != ref_sing) & ~band)[0]
    rep.info_fail = bad.tolist()
    reg = ~ref_sing & ~gpu_sing
    if kappa is None:
        kappa = np.full(B, np.inf)
        Ar = A[reg].astype(np.float64)
        Xr = ref.inverse[reg]
        kappa[reg] = np.abs(Ar).sum(2).max(1) * np.abs(Xr).sum(2).max(1)
    idx = np.nonzero(reg)[0]
    if "inverse" in gpu and gpu["inverse"] is not None:
        Xg = gpu["inverse"][idx].astype(np.float64)
        Xr = ref.inverse[idx]
        e = np.abs(Xg - Xr).max(axis=(1, 2)) / np.abs(Xr).max(axis=(1, 2))
        rep.max_inv_err = float(e.max()) if len(e) else 0.0
        ke = kappa[idx] * eps
        rep.max_inv_err_over_keps = float((e / ke).max()) if len(e) else 0.0
        flat = e <= TOL_INV[dtype]
        rep.inv_flat_fail = idx[~flat].tolist()
        rep.inv_kappa_fail = idx[~flat & ~(e <= ke)].tolist()
        if flat_only:
            rep.inv_kappa_fail = rep.inv_flat_fail
    if check_ipiv and "ipiv" in gpu:
        full = "jpiv" in gpu and getattr(ref, "jpiv", None) is not None
        for b in idx:
            ok, ex = ipiv_match(gpu["ipiv"][b], ref.ipiv[b], ref.gap[b],
                                gpu["jpiv"][b] if full else None, ref.jpiv[b] if full else None,
                                thr=tie_gap(dtype, A.shape[-1]))
            if ex and ok:
                g = first_divergence_gap(gpu["ipiv"][b], ref.ipiv[b], ref.gap[b]) if not full else 0.0
                if g is not None and g > TIE_GAP:
                    rep.ipiv_g26_exempt += 1
                    rep.ipiv_g26_items.append(int(b))
                else:
                    rep.ipiv_tie_exempt += 1
            if not ok:
                rep.ipiv_fail.append(int(b))
    if "sign" in gpu:
        numer_sing = kappa[idx] * eps >= 0.1
        sbad = (gpu["sign"][idx] != ref.sign[idx]) & ~numer_sing
        rep.sign_fail = idx[sbad].tolist()
        # singular items: sign 0
        sidx = np.nonzero(ref_sing & gpu_sing)[0]
        rep.sign_fail += sidx[gpu["sign"][sidx] != 0].tolist()
    if "logabsdet" in gpu:
        d = np.abs(gpu["logabsdet"][idx] - ref.logabsdet[idx])
        rep.max_logdet_err = float(d.max()) if len(d) else 0.0
        lim = np.maximum(TOL_INV[dtype], kappa[idx] * eps)
        rep.logdet_fail = idx[~(d <= lim)].tolist()
    if check_det and "det" in gpu:
        r = np.abs(gpu["det"][idx].astype(np.float64) - ref.det[idx]) / np.abs(ref.det[idx])
        rep.det_fail = idx[~(r <= det_rtol)].tolist()
    return rep


def assert_report(rep: Report, flat_only=False, max_kappa_fail=0):
    msg = rep.summary()
    assert not rep.info_fail, msg
    assert not rep.ipiv_fail, msg
    assert not rep.sign_fail, msg
    assert not rep.logdet_fail, msg
    assert not rep.det_fail, msg
    if flat_only:
        assert not rep.inv_flat_fail, msg
    assert len(rep.inv_kappa_fail) <= max_kappa_fail, msg

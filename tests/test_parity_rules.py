"""Host logic of the parity rules (tests/parity.py): the R3 pivot-sequence rule and its
precision-aware exemption threshold (reading G26)."""
import numpy as np

from tests.parity import TIE_GAP, ipiv_match, tie_gap


def test_tie_gap_values():
    assert tie_gap(np.float64, 32) == TIE_GAP == 1e-6
    assert tie_gap(np.float64, 8192) == 1e-6               # 8192 * 2^-53 = 9e-13
    assert tie_gap(np.float32, 32) == 32 * 2.0 ** -24      # 1.9e-6 > 1e-6
    assert tie_gap(np.float32, 8) == 1e-6                  # 4.8e-7 < 1e-6


def test_ipiv_rule():
    ref = np.arange(1, 9, dtype=np.int32)
    gap = np.full(8, 0.5)
    assert ipiv_match(ref.copy(), ref, gap) == (True, False)
    gpu = ref.copy()
    gpu[3] = 7
    assert ipiv_match(gpu, ref, gap) == (False, True)       # decided step: must match
    gap[3] = 1.064e-6                                       # C2 item 962732's step 27
    assert ipiv_match(gpu, ref, gap)[0] is False            # north-star threshold alone
    assert ipiv_match(gpu, ref, gap, thr=tie_gap(np.float32, 32))[0] is True
    assert ipiv_match(gpu, ref, gap, thr=tie_gap(np.float64, 32))[0] is False
    gpu[5] = 1                                              # later steps are not compared
    assert ipiv_match(gpu, ref, gap, thr=tie_gap(np.float32, 32))[0] is True

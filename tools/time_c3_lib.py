"""C3 timing (262,144 x 64 x 64 fp64, seed 2, tol 1e-10) from given libgjinv.so builds, with
and without ipiv (without: the two-pass K2f run), and bitwise equality of every output
requested by both calls:   python tools/time_c3_lib.py LIB [LIB ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
A = torch.from_numpy(synth.gen_c3()).cuda()
B = A.shape[0]
s = torch.cuda.current_stream().cuda_stream
ref = None
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gj_invert_batched.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    for with_ipiv in (True, False):
        X = torch.empty_like(A)
        perm = torch.empty((B, 64), dtype=torch.int32, device="cuda") if with_ipiv else None
        det = torch.empty(B, dtype=torch.float64, device="cuda")
        lad = torch.empty(B, dtype=torch.float64, device="cuda")
        sg = torch.empty(B, dtype=torch.int8, device="cuda")
        info = torch.empty(B, dtype=torch.int32, device="cuda")
        call = lambda: L.gj_invert_batched(1, 64, B, A.data_ptr(), X.data_ptr(), None if perm is None else perm.data_ptr(),
                                           lad.data_ptr(), sg.data_ptr(), det.data_ptr(), info.data_ptr(), synth.C3_TOL, s)
        for _ in range(3):
            assert call() == 0
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        outs = (X.view(torch.int64), lad.view(torch.int64), sg, det.view(torch.int64), info)
        if ref is None:
            ref = [o.clone() for o in outs]
            eq = "reference"
        else:
            eq = all(torch.equal(a, b) for a, b in zip(ref, outs))
        print(f"{path} ipiv={with_ipiv}: median {np.median(ts):.3f} ms  min {min(ts):.3f}  bitwise equal: {eq}", flush=True)

"""f4 timing (C2 batch: det-only gj_det and gj_solve_batched with 1 rhs, no ipiv) from given
libgjinv.so builds:  python tools/time_f4_lib.py LIB [LIB ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

A = torch.from_numpy(synth.gen_c2(batch=1048576)).cuda()
B = A.shape[0]
g = torch.Generator(device="cuda").manual_seed(5)
R = torch.randn((B, 32, 1), generator=g, device="cuda")
X = torch.empty_like(R)
lg = torch.empty(B, dtype=torch.float64, device="cuda")
sg = torch.empty(B, dtype=torch.int8, device="cuda")
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
s = torch.cuda.current_stream().cuda_stream
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gj_det.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
    L.gj_solve_batched.argtypes = [i32, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    for name, run in (("det", lambda: L.gj_det(0, 32, B, A.data_ptr(), lg.data_ptr(), sg.data_ptr(), None, None, None,
                                              32 * 2.0 ** -23, None, 0, s)),
                      ("solve1", lambda: L.gj_solve_batched(0, 32, 1, B, A.data_ptr(), R.data_ptr(), X.data_ptr(), None,
                                                           None, None, None, 32 * 2.0 ** -23, s))):
        for _ in range(3):
            assert run() == 0
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{path} {name}: median {np.median(ts):.3f} ms", flush=True)

"""f2 timing (full pivoting on the C2 batch, no ipiv / jpiv requested) from given libgjinv.so
builds:  python tools/time_f2_lib.py LIB [LIB ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

A = torch.from_numpy(synth.gen_c2(batch=1048576)).cuda()
X = torch.empty_like(A)
B = A.shape[0]
lg = torch.empty(B, dtype=torch.float64, device="cuda")
sg = torch.empty(B, dtype=torch.int8, device="cuda")
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
s = torch.cuda.current_stream().cuda_stream
ref = None
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gj_invert_batched_full.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    run = lambda: L.gj_invert_batched_full(0, 32, B, A.data_ptr(), X.data_ptr(), None, None, lg.data_ptr(),
                                           sg.data_ptr(), None, None, 32 * 2.0 ** -23, s)
    for _ in range(2):
        assert run() == 0
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    outs = (X.view(torch.int32).clone(), lg.clone(), sg.clone())
    eq = "reference" if ref is None else all(torch.equal(p, q) for p, q in zip(ref, outs))
    ref = ref or outs
    print(f"{path}: median {np.median(ts):.3f} ms  bitwise equal: {eq}", flush=True)

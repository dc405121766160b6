"""C2 timing of gj_invert_batched from a given libgjinv.so (A/B of build variants):
    python tools/time_c2_lib.py LIB [LIB ...]"""
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
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.gj_invert_batched.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    s = torch.cuda.current_stream()
    run = lambda: L.gj_invert_batched(0, 32, B, A.data_ptr(), X.data_ptr(), None, lg.data_ptr(), sg.data_ptr(),
                                      None, None, 32 * 2.0 ** -23, s.cuda_stream)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{path}: median {np.median(ts):.3f} ms  min {min(ts):.3f} ms", flush=True)
    if path == sys.argv[1]:
        ref = (X.clone(), lg.clone(), sg.clone())
    else:
        same = torch.equal(ref[0].view(torch.int32), X.view(torch.int32)) and torch.equal(ref[1], lg) and torch.equal(ref[2], sg)
        print(f"  bitwise equal to {sys.argv[1]}: {same}", flush=True)

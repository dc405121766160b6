"""C4 timing (one fp64 8192 gj_invert) from given libgjinv.so builds (A/B)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

import os
n = int(os.environ.get("GJ_N", "8192"))
A = torch.from_numpy(synth.gen_gaussian(n, seed=3)).cuda()
X = torch.empty_like(A)
ip = torch.empty(n, dtype=torch.int32, device="cuda")
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.gj_invert.argtypes = [i32, i32, vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
    L.gj_workspace_size.argtypes = [i32, i32, i64, i32]
    L.gj_workspace_size.restype = ctypes.c_size_t
    wb = L.gj_workspace_size(1, n, 1, 1)
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    run = lambda: L.gj_invert(1, n, A.data_ptr(), n, X.data_ptr(), n, ip.data_ptr(), None, None, None, -1.0,
                              ws.data_ptr(), wb, s.cuda_stream)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{path}: median {np.median(ts):.2f} ms  min {min(ts):.2f}", flush=True)
    if path == sys.argv[1]:
        ref = (X.clone(), ip.clone())
    else:
        d = ((X - ref[0]).abs().max() / ref[0].abs().max()).item()
        print(f"  vs {sys.argv[1]}: max rel diff {d:.3e}, ipiv equal {torch.equal(ip, ref[1])}", flush=True)
    del ws

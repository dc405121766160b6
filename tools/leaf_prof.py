import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

L = ctypes.CDLL("/tmp/leafprof/libgjinv.so")
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
L.gj_invert.argtypes = [i32, i32, vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
L.gj_workspace_size.argtypes = [i32, i32, i64, i32]
L.gj_workspace_size.restype = ctypes.c_size_t
L.gj_debug_leaf_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), i32]
names = ["-", "warp reduce", "slot write + fence + bar", "CTA pick + bulk issue", "mbarrier wait",
         "cluster pick + row read", "update"]
for dt, tdt in ((1, torch.float64), (0, torch.float32)):
    n = 8192
    A = torch.from_numpy(synth.gen_gaussian(n, seed=3)).to(tdt).cuda()
    X = torch.empty_like(A)
    ws_b = L.gj_workspace_size(dt, n, 1, 1)
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    ip = torch.empty(n, dtype=torch.int32, device="cuda")
    for rep in range(2):
        out = (ctypes.c_ulonglong * 8)()
        L.gj_debug_leaf_prof(out, 1)
        s = torch.cuda.current_stream().cuda_stream
        L.gj_invert(dt, n, A.data_ptr(), n, X.data_ptr(), n, ip.data_ptr(), None, None, None, -1.0, ws.data_ptr(), ws_b, s)
        torch.cuda.synchronize()
        L.gj_debug_leaf_prof(out, 1)
    tot = sum(out[1:7])
    print(f"{tdt} n={n}: cycles per step (thread 0, CTA 0), total {tot / n:.0f}")
    for i in range(1, 7):
        print(f"  {names[i]:28s} {out[i] / n:8.0f}  {out[i] / tot * 100:5.1f}%")
    npan = n // 128
    print(f"  per panel (us at 1.965 GHz): whole leaf kernel {out[0] / npan / 1965:8.1f}, steps {tot / npan / 1965:8.1f}, "
          f"intra-panel updates {out[7] / npan / 1965:8.1f}")

"""A/B builds of the library on the fp32 n = 32 solve (nrhs 1 and 8) and det-only runs
(C2-sized batch): median ms of each.  python tools/ab_solve.py A.so B.so ..."""
import ctypes
import sys

import torch

vp, i64, i32, dbl, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
Bt = 1 << 20
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((Bt, 32, 32), generator=g, device="cuda")
RH = {m: torch.randn((Bt, 32, m), generator=g, device="cuda") for m in (1, 8)}
X = {m: torch.empty_like(RH[m]) for m in (1, 8)}
ip = torch.empty((Bt, 32), dtype=torch.int32, device="cuda")
lg = torch.empty(Bt, dtype=torch.float64, device="cuda")
sg = torch.empty(Bt, dtype=torch.int8, device="cuda")
dt = torch.empty(Bt, dtype=torch.float32, device="cuda")
inf = torch.empty(Bt, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def med(f, reps=7):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[reps // 2]


for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gj_solve_batched.argtypes = [i32, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    L.gj_det.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, dbl, vp, sz, vp]
    row = [path]
    for m in (1, 8):
        row.append(f"solve m={m} {med(lambda: L.gj_solve_batched(0, 32, m, Bt, A.data_ptr(), RH[m].data_ptr(), X[m].data_ptr(), ip.data_ptr(), lg.data_ptr(), sg.data_ptr(), inf.data_ptr(), -1.0, s)):.3f}")
    row.append(f"det {med(lambda: L.gj_det(0, 32, Bt, A.data_ptr(), lg.data_ptr(), sg.data_ptr(), dt.data_ptr(), ip.data_ptr(), inf.data_ptr(), -1.0, None, 0, s)):.3f}")
    print("  ".join(row))

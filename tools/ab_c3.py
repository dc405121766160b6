"""A/B two builds of the library on C3 (fp64 n = 64): bitwise equality of every output and
the per-batch time of each.  python tools/ab_c3.py OLD.so NEW.so"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
A = torch.from_numpy(synth.gen_c3()).cuda()
B = A.shape[0]
s = torch.cuda.current_stream().cuda_stream
outs = []
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gj_invert_batched.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
    X = torch.empty_like(A)
    perm = torch.empty((B, 64), dtype=torch.int32, device="cuda")
    det = torch.empty(B, dtype=torch.float64, device="cuda")
    lad = torch.empty(B, dtype=torch.float64, device="cuda")
    info = torch.empty(B, dtype=torch.int32, device="cuda")
    call = lambda: L.gj_invert_batched(1, 64, B, A.data_ptr(), X.data_ptr(), perm.data_ptr(), lad.data_ptr(), None,
                                       det.data_ptr(), info.data_ptr(), synth.C3_TOL, s)
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
    ts.sort()
    print(f"{path}: median {ts[5]:.3f} ms  min {ts[0]:.3f} ms")
    outs.append((X.clone(), perm.clone(), lad.clone(), det.clone(), info.clone()))
for i in range(1, len(outs)):
    eq = all(torch.equal(a.view(torch.int64) if a.dtype == torch.float64 else a,
                         b.view(torch.int64) if b.dtype == torch.float64 else b) for a, b in zip(outs[0], outs[i]))
    print(f"{sys.argv[i + 1]} vs {sys.argv[1]}: every output bitwise equal {eq}")

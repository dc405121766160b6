"""Per-phase cycles of K2d's panel step (library built with -DGJ_K2D_PROF via tools/ab_build.sh):
    python tools/k2d_prof.py /tmp/k2dp/libgjinv.so"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

L = ctypes.CDLL(sys.argv[1])
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
L.gj_invert_batched.argtypes = [i32, i32, i64, vp, vp, vp, vp, vp, vp, vp, dbl, vp]
L.gj_debug_k2d_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), i32]
A = torch.from_numpy(synth.gen_c3()).cuda()
X = torch.empty_like(A)
B = A.shape[0]
s = torch.cuda.current_stream().cuda_stream
out = (ctypes.c_ulonglong * 8)()
L.gj_invert_batched(1, 64, B, A.data_ptr(), X.data_ptr(), None, None, None, None, None, 1e-10, s)
torch.cuda.synchronize()
L.gj_debug_k2d_prof(out, 1)
L.gj_invert_batched(1, 64, B, A.data_ptr(), X.data_ptr(), None, None, None, None, None, 1e-10, s)
torch.cuda.synchronize()
L.gj_debug_k2d_prof(out, 0)
items = (B + 148 * 4 - 1) // (148 * 4)   # CTA 0's items (grid = 4 CTAs per SM)
steps = items * 64
names = ["-", "3 reductions (fp64 key)", "pivot row shuffles", "1/p (rcp + Newton)", "row updates + bookkeeping", "record"]
tot = sum(out[1:6])
print(f"cycles per pivot step (CTA 0, warp 0): {tot / steps:.0f}")
for i in range(1, 6):
    print(f"  {names[i]:28s} {out[i] / steps:7.0f}  {out[i] / tot * 100:5.1f}%")

"""Per-panel timeline of one large-n gj_invert from a -DGJ_TIMELINE build (diagnostic):
leaf start/end and trailing-update start / last-CTA start / end, in us from the first leaf.
  python tools/timeline_large.py LIB [n]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
L = ctypes.CDLL(path)
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
L.gj_invert.argtypes = [i32, i32, vp, i64, vp, i64, vp, vp, vp, vp, dbl, vp, ctypes.c_size_t, vp]
L.gj_workspace_size.argtypes = [i32, i32, i64, i32]
L.gj_workspace_size.restype = ctypes.c_size_t
L.gj_debug_timeline.argtypes = [vp, i32]
A = torch.from_numpy(synth.gen_gaussian(n, seed=3)).cuda()
X = torch.empty_like(A)
ip = torch.empty(n, dtype=torch.int32, device="cuda")
wb = L.gj_workspace_size(1, n, 1, 1)
ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
buf = np.zeros((5, 512), dtype=np.uint64)
for rep in range(2):
    L.gj_debug_timeline(buf.ctypes.data, 1)
    L.gj_invert(1, n, A.data_ptr(), n, X.data_ptr(), n, ip.data_ptr(), None, None, None, -1.0, ws.data_ptr(), wb,
                torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    L.gj_debug_timeline(buf.ctypes.data, 0)
t0 = buf[0, 0]
npan = (n + 127) // 128
print("panel  leaf_start leaf_end  gemm_start gemm_last_cta gemm_end   (us)")
rows = []
for k in range(npan):
    r = [(int(buf[i, k]) - int(t0)) / 1e3 if buf[i, k] not in (0, 2 ** 64 - 1) else float("nan") for i in range(5)]
    rows.append(r)
    if k < 6 or k > npan - 3:
        print(f"{k:5d} {r[0]:10.1f} {r[1]:9.1f} {r[2]:10.1f} {r[4]:12.1f} {r[3]:9.1f}")
# rows: [leaf start, leaf end, gemm start, gemm end, gemm last-CTA start]
R = np.array(rows)[:, [0, 1, 2, 3, 4]]
print("leaf ms each (mean)", np.nanmean(R[:, 1] - R[:, 0]), " gemm (mean)", np.nanmean(R[:, 3] - R[:, 2]),
      " gemm last-CTA start after gemm start (mean)", np.nanmean(R[:, 4] - R[:, 2]),
      " per-panel period", np.nanmean(np.diff(R[:, 0])))

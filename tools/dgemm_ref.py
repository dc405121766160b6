"""Context numbers for the large-n path: cuBLAS DGEMM (torch.mm fp64) at the trailing-update
shape (8192 x 128 x 8064, C += A B) and at 8192^3, with the SM clock sampled during each."""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")


def clocks(fn, reps):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    mhz = sorted(float(l.split(",")[0]) for l in out if l.strip())
    return s.elapsed_time(e) / reps, (mhz[len(mhz) // 2] if mhz else None), out[-3:] if out else []


n = 8192
A = torch.randn(n, 128, dtype=torch.float64, device="cuda")
B = torch.randn(128, n - 128, dtype=torch.float64, device="cuda")
C = torch.randn(n, n - 128, dtype=torch.float64, device="cuda")
ms, mhz, tail = clocks(lambda: C.addmm_(A, B), 50)
print(f"cuBLAS DGEMM {n}x128x{n-128} (C+=AB): {ms:.3f} ms  {2*n*128*(n-128)/ms/1e9:.0f} GFLOP/s  sm_mhz~{mhz} {tail}")
X = torch.randn(n, n, dtype=torch.float64, device="cuda")
Y = torch.randn(n, n, dtype=torch.float64, device="cuda")
ms, mhz, tail = clocks(lambda: torch.mm(X, Y), 5)
print(f"cuBLAS DGEMM {n}^3: {ms:.3f} ms  {2*n**3/ms/1e9:.0f} GFLOP/s  sm_mhz~{mhz} {tail}")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402
At = torch.from_numpy(synth.gen_gaussian(n, seed=3)).cuda()
Xo = torch.empty_like(At)
ms, mhz, tail = clocks(lambda: gj.invert(At, out=Xo), 3)
print(f"gj_invert n={n}: {ms:.2f} ms  {(2*n**3-n*n)/ms/1e9:.0f} GFLOP/s  sm_mhz~{mhz} {tail}")

"""Time gj_invert_batched on BASELINE configs C1/C2/C3 inputs (device-resident, CUDA events
on the launching stream) and print matrices/s, GB/s and GFLOP/s per config."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_7962_b200 as gj  # noqa: E402
import synth  # noqa: E402

cfgs = sys.argv[1:] or ["c1", "c3"]
for c in cfgs:
    if c == "c1":
        A = synth.gen_c1()
    elif c == "c2":
        A = synth.gen_c2(batch=1048576)
    elif c == "c3":
        A = synth.gen_c3()
    B, n = A.shape[0], A.shape[1]
    At = torch.from_numpy(A).cuda()
    X = torch.empty_like(At)
    es = At.element_size()
    lg = torch.empty(B, dtype=torch.float64, device="cuda")
    sg = torch.empty(B, dtype=torch.int8, device="cuda")
    det = torch.empty(B, dtype=At.dtype, device="cuda")
    ip = torch.empty((B, n), dtype=torch.int32, device="cuda")
    info = torch.empty(B, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    tol = 1e-10 if c == "c3" else -1.0

    def run():
        st = gj.lib.gj_invert_batched(1 if es == 8 else 0, n, B, At.data_ptr(), X.data_ptr(), ip.data_ptr(), lg.data_ptr(),
                                      sg.data_ptr(), det.data_ptr(), info.data_ptr(), tol, s.cuda_stream)
        assert st == 0

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    by = B * (2 * n * n * es + n * 4 + 8 + 1 + es + 4)
    fl = B * (2 * n ** 3 - n ** 2)
    print(f"{c}: B={B} n={n} {ms:.3f} ms  {B / ms * 1e3:.3e} mat/s  {by / ms / 1e6:.0f} GB/s  {fl / ms / 1e9:.0f} GFLOP/s"
          f"  singular={int((info.cpu() != 0).sum())}", flush=True)

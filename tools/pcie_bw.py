"""Raw pinned-host <-> device copy bandwidth (context for the e2e number): H2D alone, D2H
alone, both at once on two streams."""
import time
import torch
n = 1 << 30  # 1 GiB (as fp32 elements * 4 = 4 GiB)
h1 = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t0
gb = n * 4 / 1e9
th = t(lambda: d1.copy_(h1, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
tb = t(both)
print(f"H2D {gb / th:.1f} GB/s  D2H {gb / td:.1f} GB/s  both {2 * gb / tb:.1f} GB/s total")

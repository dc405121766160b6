"""C2 item 962732 (the one item of the 1,048,576 whose GPU pivot sequence leaves the
long-double oracle's at a step with gap > 1e-6): run plain sequential partial-pivoting
Gauss–Jordan (the listing's order: divide the pivot row, subtract multiples) in fp32, fp64
and long double and print each one's pivot at the first step where they can differ, with
the step's relative gap in each precision.  Evidence for reading G26."""
import numpy as np

ITEM = 962732
rng = np.random.default_rng(1)
for s in range(0, ITEM // 65536 + 1):
    ch = rng.standard_normal((65536, 32, 32), dtype=np.float32)
A0 = ch[ITEM - (ITEM // 65536) * 65536]


def gj(A, dt):
    a = np.concatenate([A.astype(dt), np.eye(32, dtype=dt)], axis=1)
    piv, gaps = [], []
    for k in range(32):
        col = np.abs(a[k:, k])
        q = k + int(np.argmax(col))
        srt = np.sort(col)[::-1]
        gaps.append(float((srt[0] - srt[1]) / srt[0]) if len(srt) > 1 else 1.0)
        piv.append(q)
        a[[k, q]] = a[[q, k]]
        a[k] = a[k] / a[k, k]
        for i in range(32):
            if i != k:
                a[i] = a[i] - a[i, k] * a[k]
    return piv, gaps


res = {name: gj(A0, dt) for name, dt in (("fp32", np.float32), ("fp64", np.float64), ("longdouble", np.longdouble))}
for name, (p, g) in res.items():
    print(f"{name:10s} pivots 25..29: {p[25:30]}  gap at 27: {g[27]:.3e}")

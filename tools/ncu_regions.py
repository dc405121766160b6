"""Split executed instructions of an ncu SASS dump into prologue / loop / epilogue
around the CREDUX (pivot-search) region; per-item normalisation by argv[2]."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    try: ex = int(r[idx['Instructions Executed']] or 0)
    except ValueError: continue
    data.append((int(r[idx['Address']], 16), r[idx['Source']].strip(), ex))
cr = [a for a, s, e in data if 'CREDUX' in s and e > 0]
lo, hi = (min(cr), max(cr)) if cr else (0, 0)
def op(s):
    t = s.split()
    return (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
for name, sel in (("prologue", lambda a: a < lo - 0x200), ("loop", lambda a: lo - 0x200 <= a <= hi + 0x800), ("epilogue", lambda a: a > hi + 0x800)):
    c = Counter(); tot = 0
    for a, s, e in data:
        if sel(a): c[op(s)] += e; tot += e
    print(f"{name}: {tot / norm:.1f}  " + ", ".join(f"{k} {v / norm:.1f}" for k, v in c.most_common(12)))

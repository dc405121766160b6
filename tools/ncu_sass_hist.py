"""Opcode histogram (executed warp instructions, stall samples, shared wavefronts) of an
ncu `--page source --csv --print-source sass` dump, normalised per unit (argv[2])."""
import csv, sys
from collections import Counter, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
ex = Counter(); st = Counter(); wf = Counter(); tot = 0; tst = 0
for r in rows[2:]:
    if len(r) < len(hdr): continue
    s = r[idx['Source']].strip()
    t = s.split()
    if not t: continue
    o = t[1] if t[0].startswith('@') else t[0]
    o = o.rstrip(';')
    try:
        e = int(r[idx['Instructions Executed']] or 0); smp = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
        w = int(r[idx['L1 Wavefronts Shared']] or 0)
    except ValueError:
        continue
    ex[o] += e; st[o] += smp; wf[o] += w; tot += e; tst += smp
print(f"total instr/unit {tot / norm:.1f}; stall samples {tst}")
for k, v in ex.most_common(40):
    print(f"{k:28s} instr/unit {v / norm:8.1f}  samples {100.0 * st[k] / max(tst, 1):5.1f}%  smem wf/unit {wf[k] / norm:7.1f}")

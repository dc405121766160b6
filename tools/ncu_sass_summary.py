"""Summarise an `ncu --page source --csv --print-source=sass` dump: stall reasons and
instruction mix weighted by execution count (used to write profiles/*.md)."""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
stalls = Counter()
mix = Counter()
total_exec = 0
smem_excess = 0
smem_total = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[idx["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        ex = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    mix[op] += ex
    total_exec += ex
    for c in stall_cols:
        try:
            stalls[c] += int(r[idx[c]] or 0)
        except ValueError:
            pass
    try:
        smem_excess += int(r[idx["L1 Wavefronts Shared Excessive"]] or 0)
        smem_total += int(r[idx["L1 Wavefronts Shared"]] or 0)
    except (ValueError, KeyError):
        pass
print(f"executed warp instructions: {total_exec}")
print("instruction mix (top 25):")
for op, c in mix.most_common(25):
    print(f"  {op:14s} {c:14d} {100.0 * c / total_exec:6.2f}%")
ts = sum(stalls.values())
print("stall samples (top 12):")
for s, c in stalls.most_common(12):
    print(f"  {s:28s} {c:10d} {100.0 * c / max(ts, 1):6.2f}%")
print(f"shared wavefronts: {smem_total}, excessive: {smem_excess}")

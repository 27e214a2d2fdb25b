"""Summarise an ncu --page source --print-source sass CSV: executed
instructions per opcode and the hottest stall sites.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > s.csv
    python tools/sass_hist.py s.csv [nodes]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
nodes = float(sys.argv[2]) if len(sys.argv) > 2 else None
ops = Counter()
tot = 0
stalls = []
for d in data:
    src = d["Source"].strip()
    n = float(d["Instructions Executed"] or 0)
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    tot += n
    stalls.append((float(d["Warp Stall Sampling (All Samples)"] or 0), d["Address"], src, n))
print(f"total warp-instructions {tot:.4g}" + (f"  thread-instr/node {32 * tot / nodes:.1f}" if nodes else ""))
for op, n in ops.most_common(25):
    print(f"  {op:10s} {n:12.4g} {100 * n / tot:5.1f}%" + (f"  {32 * n / nodes:6.2f}/node" if nodes else ""))
print("hottest stall sites:")
for s, a, src, n in sorted(stalls, reverse=True)[:25]:
    print(f"  {s:7.0f}  {src[:70]}")

"""Attribute executed SASS instructions of chosen opcode classes to CUDA
source lines (ncu source page, cuda+sass and sass-only CSV exports).

    ncu -i rep --page source --csv --print-source sass > s.csv
    ncu -i rep --page source --csv --print-source cuda,sass > cs.csv
    python tools/op_by_line.py s.csv cs.csv NODES PREFIX[,PREFIX...] [top]
"""
import csv
import re
import sys
from collections import defaultdict

s_csv, cs_csv, nodes = sys.argv[1], sys.argv[2], float(sys.argv[3])
prefixes = tuple(sys.argv[4].split(","))
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
rows = list(csv.reader(open(s_csv, encoding="utf-8", errors="replace")))
hdr = rows[1]
cnt = {}
for r in rows[2:]:
    if len(r) == len(hdr):
        d = dict(zip(hdr, r))
        cnt[d["Address"]] = (float(d["Instructions Executed"] or 0), d["Source"].strip())
line_of = {}
fname, cur = None, None
for r in csv.reader(open(cs_csv, encoding="utf-8", errors="replace")):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 4 and r[0] not in ("", "Line No"):
        cur = f"{fname}:{r[0]} {r[1][:70]}"
    elif len(r) >= 4 and r[0] == "" and r[2].startswith("0x"):
        line_of[r[2]] = cur
agg = defaultdict(float)
for addr, (n, src) in cnt.items():
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    if op.startswith(prefixes):
        agg[line_of.get(addr, "?")] += n * 32 / nodes
tot = sum(agg.values())
print(f"total {tot:.2f}/node")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:6.2f}  {k}")

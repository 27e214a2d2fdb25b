"""Per CUDA source line: executed instructions by opcode class and stall
samples, from `ncu --page source --csv --print-source cuda,sass`.

    python tools/line_ops.py src.csv nodes [top]
"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
nodes = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, line, src = None, None, None
per = defaultdict(Counter)
stall = Counter()
text = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Line No", "Function Name"):
        continue
    if r[0] != "":
        line = (fname, r[0])
        text[line] = r[1][:70]
        continue
    if len(r) < 8 or line is None:
        continue
    s = r[3].strip()
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    op = op.split(".")[0]
    try:
        n = float(r[7] or 0)
    except ValueError:
        continue
    per[line][op] += n
    stall[line] += float(r[4]) if r[4] not in ("", "-") else 0.0
tot = {k: sum(v.values()) for k, v in per.items()}
ts = sum(stall.values()) or 1
for k in sorted(tot, key=lambda k: -tot[k])[:top]:
    c = per[k]
    fp = c["DFMA"] + c["DMUL"] + c["DADD"]
    print(f"{k[0][:12]}:{k[1]:>4} {32*tot[k]/nodes:6.2f}/node fp64 {32*fp/nodes:5.2f} "
          f"(M{32*c['DMUL']/nodes:.2f}) st {100*stall[k]/ts:4.1f}% | {text[k]}")

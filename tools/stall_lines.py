"""Top CUDA source lines by a given stall reason (ncu source page).

    python tools/stall_lines.py rep.ncu-rep stall_long_sb [top]
"""
import csv
import io
import subprocess
import sys

rep, reason = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, hdr, out = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ci = hdr.index(reason)
        continue
    if hdr and len(r) == len(hdr) and r[0] != "":
        try:
            out.append((float(r[ci] or 0), fname, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
for n, f, l, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * n / tot:5.1f}% {f[:14]}:{l:>4} {src}")

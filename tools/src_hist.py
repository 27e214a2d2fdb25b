"""Per-CUDA-source-line executed instructions from an ncu report.

    python tools/src_hist.py rep.ncu-rep [nodes] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nodes = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
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
        continue
    if hdr and len(r) == len(hdr) and r[0] != "":
        try:
            n = float(r[7] or 0)
            st = float(r[4] or 0)
        except ValueError:
            continue
        out.append((n, fname, r[0], r[1][:90], st))
tot = sum(o[0] for o in out)
print(f"total {tot:.4g} warp-instr = {32 * tot / nodes:.1f} thread-instr/node")
for n, f, l, src, st in sorted(out, reverse=True)[:top]:
    print(f"{32 * n / nodes:6.2f}/node stall{st:6.0f} {f[:14]}:{l:>4} {src}")

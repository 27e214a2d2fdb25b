"""Shared-memory wavefronts and executed instructions per opcode from an
`ncu --page source --csv --print-source sass` export (k_micro32 profiles).

    python tools/wf_by_op.py base.csv new.csv [nodes]
"""
import collections
import csv
import sys


def agg(path):
    rows = list(csv.reader(open(path, encoding="utf-8", errors="replace")))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    wf, n = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        src = r[ix["Source"]].strip().split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        n[op] += float(r[ix["Instructions Executed"]] or 0)
        wf[op] += float(r[ix["L1 Wavefronts Shared"]] or 0)
    return wf, n


nodes = float(sys.argv[3]) if len(sys.argv) > 3 else 67108864.0
A = [agg(p) for p in sys.argv[1:3]]
ops = sorted(set(A[0][1]) | set(A[1][1]), key=lambda o: -(A[0][0][o] + A[1][0][o] + 1e-9 * (A[0][1][o] + A[1][1][o])))
print(f"{'opcode':28s} {'wf/node A':>10s} {'wf/node B':>10s} {'thr-ins/node A':>15s} {'B':>8s}")
tot = [0, 0, 0, 0]
for o in ops:
    a_wf, b_wf = A[0][0][o] / nodes, A[1][0][o] / nodes
    a_n, b_n = A[0][1][o] * 32 / nodes, A[1][1][o] * 32 / nodes
    tot = [tot[0] + a_wf, tot[1] + b_wf, tot[2] + a_n, tot[3] + b_n]
    if max(a_wf, b_wf) > 0.002 or abs(a_n - b_n) > 0.3:
        print(f"{o:28s} {a_wf:10.3f} {b_wf:10.3f} {a_n:15.2f} {b_n:8.2f}")
print(f"{'TOTAL':28s} {tot[0]:10.3f} {tot[1]:10.3f} {tot[2]:15.2f} {tot[3]:8.2f}")

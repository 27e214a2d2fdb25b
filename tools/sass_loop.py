"""Static opcode mix of a kernel's steady row loop (the longest loop that is
not the outer general-body loop: pick by rank among backward branches).

    cuobjdump -sass -fun <mangled> obj.o | python tools/sass_loop.py [lo hi]
"""
import re
import sys
from collections import Counter

ins = []
for line in sys.stdin:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
loops = []
for a, t in ins:
    m2 = re.search(r"BRA.*0x([0-9a-f]+)", t)
    if m2 and int(m2.group(1), 16) < a:
        loops.append((int(m2.group(1), 16), a))
if len(sys.argv) > 2:
    best = (int(sys.argv[1], 0), int(sys.argv[2], 0))
else:
    # the steady loop: the longest loop that contains no other loop longer than 64 instructions
    def inner(l):
        return [m for m in loops if m != l and l[0] <= m[0] and m[1] <= l[1] and m[1] - m[0] > 64 * 16]
    cand = [l for l in loops if not inner(l)]
    best = max(cand, key=lambda l: l[1] - l[0])
body = [t for a, t in ins if best[0] <= a <= best[1]]
ops = Counter()
for t in body:
    w = t.split()
    op = w[1] if w[0].startswith("@") else w[0]
    parts = op.split(".")
    key = parts[0]
    if key in ("LDS", "STS", "LDG", "STG") and len(parts) > 1:
        key += "." + parts[-1]
    ops[key] += 1
print(f"loop {best[0]:#x}..{best[1]:#x}: {len(body)} static instructions")
f64 = sum(n for o, n in ops.items() if o in ("DFMA", "DMUL", "DADD"))
print(f"fp64 {f64}")
for o, n in ops.most_common(40):
    print(f"  {o:12s} {n}")

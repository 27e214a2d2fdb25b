"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)
into per-kernel counts, mean durations and shares of this library's time.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline
    python tools/launch_list.py launches.csv
"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1], errors="replace")) if len(r) > 5]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("mm2d::", "")
    agg[name].append(float(r[vi].replace(",", "")))
ours = {k: v for k, v in agg.items() if "k_" in k}
tot = sum(sum(v) for v in ours.values()) or 1.0
print(f"{'kernel':44s}{'launches':>9s}{'mean_ns':>12s}{'share':>8s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = sum(v) / tot if k in ours else float("nan")
    print(f"{k[:44]:44s}{len(v):9d}{sum(v) / len(v):12.0f}{share:8.3f}")

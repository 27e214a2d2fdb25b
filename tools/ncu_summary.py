"""Key metrics + stall reasons of one kernel in an ncu report.

    python tools/ncu_summary.py rep.ncu-rep
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "L2 Hit Rate",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Dynamic Shared Memory Per Block", "Executed Instructions", "L1/TEX Hit Rate",
        "Mem Pipes Busy", "Shared Memory Throughput"]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:38s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, v = rr[0], rr[2]
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x or 0)) for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
tot = sum(x for _, x in st) or 1
print("stalls:", ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in sorted(st, key=lambda t: -t[1])[:9]))
for k, x in zip(h, v):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
             "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
             "smsp__inst_executed_op_shared_ld.sum"):
        print(k, x)

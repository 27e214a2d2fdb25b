"""Side-by-side key metrics of k_micro32 from ncu --set full reports.

    python tools/ncu_cmp.py a.ncu-rep b.ncu-rep ...
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wf %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex thru % (active)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank conflicts"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed.sum", "warp instr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps/sched"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("smsp__average_warp_latency_issue_stalled_short_scoreboard", "stall short_sb"),
    ("smsp__average_warp_latency_issue_stalled_wait", "stall wait"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
    ("smsp__average_warp_latency_issue_stalled_mio_throttle", "stall mio_throttle"),
    ("smsp__average_warp_latency_issue_stalled_lg_throttle", "stall lg_throttle"),
    ("smsp__average_warp_latency_issue_stalled_math_pipe_throttle", "stall math_pipe"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_sb"),
    ("smsp__average_warp_latency_issue_stalled_dispatch_stall", "stall dispatch"),
    ("smsp__average_warp_latency_issue_stalled_not_selected", "stall not_selected"),
    ("smsp__average_warp_latency_issue_stalled_selected", "stall selected"),
    ("smsp__average_warp_latency_issue_stalled_no_instruction", "stall no_inst"),
    ("smsp__average_warp_latency_issue_stalled_tex_throttle", "stall tex"),
    ("smsp__average_warp_latency_issue_stalled_membar", "stall membar"),
    ("smsp__average_warp_latency_issue_stalled_sleeping", "stall sleeping"),
    ("smsp__average_warp_latency_issue_stalled_branch_resolving", "stall branch"),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        if any("k_micro32" in c for c in r):
            return dict(zip(h, r))
    return {}


reps = [load(r) for r in sys.argv[1:]]
print(f"{'':28s}" + "".join(f"{a.split('/')[-1][:22]:>24s}" for a in sys.argv[1:]))
for k, name in KEYS:
    vals = []
    for d in reps:
        v = d.get(k, "")
        if v == "":
            # try a prefix match (metric suffixes differ between versions)
            cands = [kk for kk in d if kk.startswith(k)]
            v = d[cands[0]] if cands else "-"
        vals.append(v)
    print(f"{name:28s}" + "".join(f"{v:>24s}" for v in vals))

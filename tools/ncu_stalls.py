"""Summarise an ncu --set full report of the grid kernel: duration, pipes,
issue, occupancy and the warp-stall sample breakdown.
    python tools/ncu_stalls.py gpurun_out/prof_c2_fp32.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = {a: (c, b) for a, b, c in zip(h, u, v)}
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_write.sum.per_second"]
for k in keys:
    if k in d:
        print(f"{k:62s} {d[k][0]:>16s} {d[k][1]}")
st = {a.split("stalled_")[1]: float(c[0].replace(",", "")) for a, c in d.items()
      if a.startswith("smsp__pcsamp_warps_issue_stalled_") and not a.endswith("not_issued")}
tot = sum(st.values()) or 1.0
print("stall samples:", "  ".join(f"{k}:{100 * x / tot:.1f}%" for k, x in
                                   sorted(st.items(), key=lambda kv: -kv[1]) if x))

"""Summarise an .ncu-rep: key section metrics + warp-stall samples (run here, not on the box)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Achieved Occupancy", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block")
for row in csv.reader(io.StringIO(det)):
    if len(row) > 14 and row[12] in keys:
        print(f"{row[12]:38s} {row[14]:>14s} {row[13]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
st = []
for k, x in zip(h, v):
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(a for a, _ in st) or 1
print("stall samples:", ", ".join(f"{k} {100 * a / tot:.0f}%" for a, k in sorted(st, reverse=True)[:8]))
for k, x in zip(h, v):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum", "smsp__inst_executed.sum",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
             "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
             "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
             "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"):
        print(k, x)

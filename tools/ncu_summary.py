"""Summarise an ncu report (details + stall reasons) into a compact text block for profiles/."""
import csv
import subprocess
import sys

rep = sys.argv[1]
det = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout.splitlines()))
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))
h = det[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Dynamic Shared Memory Per Block", "L1/TEX Hit Rate"]
seen = {}
for r in det[1:]:
    if r[mi] in want and r[mi] not in seen:
        seen[r[mi]] = f"{r[vi]} {r[ui]}"
print(f"kernel: {det[1][ki]}")
for k in want:
    if k in seen:
        print(f"  {k}: {seen[k]}")
hdr, vals = raw[0], raw[2]
pick = {}
for i, k in enumerate(hdr):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            pick[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
        except ValueError:
            pass
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
             "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
        print(f"  {k}: {vals[i]} {raw[1][i]}")
tot = sum(pick.values()) or 1
print("  stall samples (top):", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(pick.items(), key=lambda x: -x[1])[:7]))

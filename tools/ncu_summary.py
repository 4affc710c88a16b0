"""Summarise an ncu report: key details + per-source-line instruction shares.
Usage: python tools/ncu_summary.py report.ncu-rep [top_lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
KEYS = ("Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Grid Size",
        "Dynamic Shared Memory Per Block", "DRAM Throughput", "L1/TEX Hit Rate")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in KEYS:
        print(f"{d['Metric Name']:42s} {d['Metric Value']:>14s} {d.get('Metric Unit', '')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h, u, v = rr[0], rr[1], rr[2]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                 "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum"):
        if name in h:
            i = h.index(name)
            print(f"{name:60s} {v[i]:>16s} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ie = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
lines, tot, stot = [], 0, 0
for r in rows[hi + 1:]:
    if r and r[0].isdigit():
        n = int(r[ie]) if r[ie].isdigit() else 0
        s = int(r[st]) if r[st].isdigit() else 0
        lines.append((n, s, int(r[0]), r[1][:80]))
        tot += n
        stot += s
print("instructions (warp-level, source lines):", tot)
for n, s, ln, txt in sorted(lines, reverse=True)[:top]:
    print(f"{100 * n / tot:5.1f}% inst {100 * s / max(stot, 1):5.1f}% stall  L{ln:4d} {txt}")

"""Markdown summary of an ncu report (one section per profiled launch) and
of an ncu launch list (--metrics gpu__time_duration.sum CSV).

  python tools/ncu_report.py full  report.ncu-rep  > profiles/rN_<name>.md
  python tools/ncu_report.py launches launches.csv > profiles/rN_launches.md
"""
import collections
import csv
import io
import subprocess
import sys

DETAILS = ("Duration", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "No Eligible",
           "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
           "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
           "Avg. Not Predicated Off Threads Per Warp", "Executed Instructions",
           "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Grid Size",
           "Block Size", "Dynamic Shared Memory Per Block", "DRAM Throughput", "L1/TEX Hit Rate",
           "L2 Hit Rate")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
       "launch__registers_per_thread")


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def full(rep):
    det = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    h = det[0]
    per = collections.OrderedDict()
    for r in det[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        if d["Metric Name"] in DETAILS:
            per.setdefault(key, {})[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}"
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    rh, units = raw[0], raw[1]
    rawper = {}
    for r in raw[2:]:
        d = dict(zip(rh, r))
        rawper[(d["ID"], d["Kernel Name"])] = {m: f"{d.get(m, '')} {units[rh.index(m)]}"
                                               for m in RAW if m in rh}
    print(f"# ncu --set full summary of `{rep.split('/')[-1]}`\n")
    for key, vals in per.items():
        print(f"## launch {key[0]}: `{key[1][:110]}`\n")
        print("| metric | value |\n|---|---|")
        for m in DETAILS:
            if m in vals:
                print(f"| {m} | {vals[m]} |")
        for m, v in rawper.get(key, {}).items():
            print(f"| {m} | {v} |")
        print()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[ki]].append(float(r[vi]))
        except ValueError:
            pass
    tot = sum(sum(v) for v in agg.values())
    print("| launches | total us | share | avg us | kernel |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {len(v)} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% | "
              f"{sum(v) / len(v) / 1e3:.1f} | `{k[:90]}` |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])

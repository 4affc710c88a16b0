"""Executed-instruction mix by SASS opcode of one kernel in an ncu report
(the `--page source --print-source=sass` view).
Usage: python tools/ncu_sass_mix.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(r for r in rows if "Instructions Executed" in r)
si, ie = hdr.index("Source"), hdr.index("Instructions Executed")
mix = collections.Counter()
tot = 0
for r in rows:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    ins = re.sub(r"^\s*@!?U?P[0-9T]\s+", "", r[si]).strip()
    op = ins.split(" ")[0].rstrip(";")
    base = op.split(".")[0]
    n = int(r[ie])
    mix[base] += n
    tot += n
print(f"warp instructions executed: {tot}")
for op, n in mix.most_common(top):
    print(f"{100.0 * n / tot:6.2f}%  {op}")

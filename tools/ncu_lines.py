"""Per-source-line thread-instruction shares of one kernel in an ncu report.
Usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
out, tw, tt, fname = [], 0, 0, ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if "Instructions Executed" in r:
        hdr = r
        ie, ti = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and r and r[0].isdigit():
        try:  # source lines with unescaped quotes (inline asm) break the CSV
            w = int(r[ie] or 0)
            t = int(r[ti] or 0)
        except (ValueError, IndexError):
            continue
        s = int(r[st] or 0) if r[st].isdigit() else 0
        tw += w
        tt += t
        if w:
            out.append((t, w, s, f"{fname}:{r[0]}", r[1][:70]))
print(f"warp-inst {tw}  thread-inst {tt}  avg lanes {tt / max(tw, 1):.1f}")
st_tot = sum(o[2] for o in out) or 1
for t, w, s, loc, txt in sorted(out, reverse=True)[:top]:
    print(f"{100 * t / tt:5.1f}% thr {100 * s / st_tot:5.1f}% stall lanes {t / w:4.1f} {loc:22s} {txt}")

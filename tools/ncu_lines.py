"""Per-source-line instructions and stall samples of one kernel in an ncu
report: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows, fname = [], ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie, iw = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] and r[0] != "Function Name" and r[2] == "-":
        try:
            rows.append((float(r[ie] or 0), float(r[iw] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except (ValueError, IndexError, NameError):
            pass
ti = sum(x[0] for x in rows) or 1
tw = sum(x[1] for x in rows) or 1
for e, w, loc, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100 * e / ti:5.1f}% inst {100 * w / tw:5.1f}% stall  {loc:22s} {src}")

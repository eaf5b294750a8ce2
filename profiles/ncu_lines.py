"""Top source lines of an ncu report by executed warp-instructions.
Usage: python profiles/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
path, rows = None, []
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1].split("/")[-1]
        continue
    if rec[0] in ("Function Name", "Line No") or len(rec) < 8 or rec[2] != "-":
        continue
    try:
        samp = float(rec[4] or 0); inst = float(rec[7] or 0); ln = int(rec[0])
    except ValueError:
        continue
    rows.append((inst, samp, path, ln, rec[1].strip()[:90]))
ti = sum(r[0] for r in rows) or 1
ts = sum(r[1] for r in rows) or 1
for inst, samp, path, ln, txt in sorted(rows, reverse=True)[:n]:
    print(f"{100*inst/ti:5.2f}% i {100*samp/ts:5.2f}% s  {path}:{ln:<5d} {txt}")

"""Summarise an ncu report per CUDA source line (warp-stall samples and
executed warp instructions), from the `cuda,sass` source view.

Usage: python profiles/ncu_source_summary.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
path = None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1].split("/")[-1]
        continue
    if rec[0] in ("Function Name", "Line No"):
        continue
    if len(rec) < 8 or rec[2] != "-":
        continue  # cuda-line summary rows have '-' in the SASS address column
    try:
        samp = float(rec[4] or 0)
        inst = float(rec[7] or 0)
    except ValueError:
        continue
    if samp or inst:
        rows.append((samp, inst, path, rec[0], rec[1].strip()[:88]))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"total stall samples {tot_s:.0f}; executed warp-instructions {tot_i:.3e}")
for samp, inst, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * samp / tot_s:5.1f}% smp {100 * inst / tot_i:5.1f}% ins  {f}:{ln:>4}  {src}")

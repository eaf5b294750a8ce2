"""Warp-stall breakdown (pc-sampling) and headline metrics of an ncu report.
Usage: python profiles/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(h, v))


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


items = [(k, num(d[k])) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_")
         and not k.endswith("not_issued") and num(d[k]) is not None]
tot = sum(x for _, x in items) or 1
for k, x in sorted(items, key=lambda kv: -kv[1])[:10]:
    print(f"stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")
for k in ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    if k in d:
        print(f"{k:64s} {d[k]}")

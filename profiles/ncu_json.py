"""Write profiles/pair_kernel_ncu.json from pair-kernel ncu captures.

Usage: python profiles/ncu_json.py --hash H C4=profiles/pair_kernel_C4_r2.ncu-rep[:n:sims] ...

H is the libstk source hash of the build that was profiled
(paper_1912_04753_b200.build.source_hash(), written next to the capture by
tools/gpu_round.sh).  bench.py reports these per-launch figures as
roofline.traffic / roofline.hw / roofline.issue only when H equals the hash of
the build it runs (a stale capture is never reported)."""
import csv
import io
import json
import os
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active",
    "smsp__inst_executed.sum": "warp_instructions",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6,
         "%": 0.01, "inst": 1}

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pair_kernel_ncu.json")
try:
    out = json.load(open(path))
except Exception:
    out = {}
args = sys.argv[1:]
src_hash = None
if args[:1] == ["--hash"]:
    src_hash, args = args[1], args[2:]
for arg in args:
    cfg, rep = arg.split("=", 1)
    n = sims = None
    if rep.count(":") == 2:
        rep, n, sims = rep.split(":")
        n, sims = int(n), int(sims)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    rec = {"capture": f"profiles/{os.path.basename(rep)} (ncu --set full --clock-control none)",
           "kernel": vals[head.index("Kernel Name")], "src_hash": src_hash, "n": n,
           "sims": sims}
    for i, name in enumerate(head):
        if name in WANT and WANT[name] not in rec and vals[i].strip():
            v = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
            rec[WANT[name]] = round(v) if WANT[name].startswith(("dram", "warp_inst")) else round(v, 6)
    # SASS-counted FP64 thread-instructions (DADD + DMUL + DFMA) per launch
    per_cycle = 0.0
    for op in ("dadd", "dmul", "dfma"):
        k = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
        if k in head and vals[head.index(k)].strip():
            per_cycle += float(vals[head.index(k)].replace(",", ""))
    if "sm__cycles_elapsed.avg" in head:
        rec["fp64_thread_instructions"] = round(
            per_cycle * float(vals[head.index("sm__cycles_elapsed.avg")].replace(",", "")))
    out[cfg] = rec
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))

"""Instruction / stall-sample share per code region of the pair kernel.
Usage: python profiles/ncu_regions.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
path = None
agg = {}
src = open("paper_1912_04753_b200/csrc/stk_kernels.cu").read().splitlines()
dev = open("paper_1912_04753_b200/csrc/stk_device.cuh").read().splitlines()
def region(path, ln):
    if path == "stk_device.cuh":
        for k in range(ln - 1, -1, -1):
            line = dev[k]
            if line.startswith("__device__"):
                name = line.split("(")[0].split()[-1]
                if name in ("rect_single_edge_weight",):
                    return "arc weight: closed form"
                if name in ("fast_atan2",):
                    return "arc weight: atan2"
                if name in ("fixed52_minus_one",):
                    return "arc term (fixed point)"
                return "arc weight: general (" + name + ")"
        return "arc weight: other"
    if path != "stk_kernels.cu":
        return "intrinsics " + path
    # find the enclosing function by scanning upward for a marker
    for k in range(ln - 1, -1, -1):
        line = src[k]
        if "void drain_main(" in line or "void drain_general(" in line or "void add_arc_term(" in line:
            return "arc drain (" + line.split("(")[0].split()[-1] + ")"
        if "for (int k = kc; k < kend; ++k)" in line or "for (int k = 0; k < m; ++k)" in line or "for (uint32_t j0 = rb; j0 < re; j0 += 32)" in line:
            return "candidate/bin loop"
        if "flush the CTA histogram" in line:
            return "flush"
        if "auto chunk = [&]" in line:
            return "chunk setup (per tile)"
        if "new tile: map the lanes to their rows" in line:
            return "tile start + neighbour load"
        if "the single drain site" in line:
            return "drain dispatch + ring compaction"
        if "stage the item's centers" in line:
            return "item setup (rows, centers)"
        if "__global__" in line:
            return "kernel prologue / task loop"
    return "other"
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
    key = region(path, ln)
    a = agg.setdefault(key, [0, 0]); a[0] += samp; a[1] += inst
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:36s} samples {100*v[0]/ts:5.1f}%  instr {100*v[1]/ti:5.1f}%  ({v[1]:.3e} warp-instr)")

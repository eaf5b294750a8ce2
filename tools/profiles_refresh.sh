#!/bin/bash
# Copy one tools/gpu_round.sh session from gpurun_out/ into profiles/ (tracked):
#   bash tools/profiles_refresh.sh r2f
# The ncu captures are stamped with the session's libstk source hash, so
# bench.py reports roofline.hw / issue / traffic only for that very build.
set -e
tag=$1; g=gpurun_out
hash=$(cat $g/src_hash_$tag.txt)
for c in C1 C2 C3 C5 C5obs; do [ -s $g/bench_${c}_$tag.json ] && cp $g/bench_${c}_$tag.json profiles/bench_${c}_r2.json; done
cp $g/bench_$tag.json profiles/bench_r2.json
cp $g/bench_ref_$tag.json profiles/bench_ref_r2.json
cp $g/launches_$tag.csv profiles/launches_r2.csv
cp $g/pytest_gpu_$tag.log profiles/pytest_gpu_r2.log
cp $g/smoke_$tag.log profiles/smoke_r2.log
[ -s $g/perm_par_$tag.json ] && cp $g/perm_par_$tag.json profiles/perm_par_r2.json
git rm -q --cached profiles/pair_kernel_C4_r2*.ncu-rep profiles/pair_kernel_C2_r2*.ncu-rep 2>/dev/null || true
rm -f profiles/pair_kernel_C4_r2*.ncu-rep profiles/pair_kernel_C2_r2*.ncu-rep
cp $g/pair_kernel_C4_$tag.ncu-rep $g/pair_kernel_C2_$tag.ncu-rep profiles/
python profiles/ncu_json.py --hash $hash C4=profiles/pair_kernel_C4_$tag.ncu-rep C2=profiles/pair_kernel_C2_$tag.ncu-rep > /dev/null
python profiles/ncu_lines.py profiles/pair_kernel_C4_$tag.ncu-rep 30 > profiles/pair_kernel_C4_r2_lines.txt
python profiles/ncu_stalls.py profiles/pair_kernel_C4_$tag.ncu-rep > profiles/pair_kernel_C4_r2_stalls.txt
echo "profiles/ refreshed from session $tag (build $hash)"

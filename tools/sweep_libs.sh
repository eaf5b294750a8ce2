# A/B of library variants (tools/variants.py) on one box:
#   bash tools/sweep_libs.sh "C4 C2" base v1 v2 ...   (base = the in-tree libstk.so)
out=gpurun_out; mkdir -p $out
cfgs=$1; shift
for rep in 1 2; do
for name in "$@"; do
  lib=scratch/lib_$name.so; [ "$name" = base ] && lib=paper_1912_04753_b200/libstk.so
  for cfg in $cfgs; do
    STK_LIB_PATH=$lib timeout 400 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > $out/sw_${cfg}_${name}_$rep.json 2>&1
    echo "$rep $cfg $name: $(tail -1 $out/sw_${cfg}_${name}_$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms kernel", round(d["roofline"]["kernel_ms_per_step"],2))' 2>&1)"
  done
done
done

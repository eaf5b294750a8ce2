# Knob sweep: one bench line per env setting (experiments only).
#   bash tools/sweep.sh C2 "X=0" "STK_TIME_RADIUS=3" ...
out=gpurun_out; mkdir -p $out
cfg=${1:-C2}; shift
for setting in "$@"; do
  name=$(echo "$setting" | tr ' =/.' '____')
  env $setting timeout 400 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline $BENCH_EXTRA > $out/sweep_${cfg}_$name.json 2>&1
  echo "$cfg $setting: $(tail -1 $out/sweep_${cfg}_$name.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms", d["roofline"]["kernel_ms_per_step"])' 2>&1)"
done

# Stencil-geometry sweep: bench lines for env knob settings (experiments only).
out=gpurun_out; mkdir -p $out
cfg=${1:-C2}; shift
for setting in "$@"; do
  env $setting timeout 400 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > $out/sweep_${cfg}_${setting//[ =]/_}.json 2>&1
  echo "$cfg $setting: $(tail -1 $out/sweep_${cfg}_${setting//[ =]/_}.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms", d["roofline"]["kernel_ms_per_step"])' 2>&1)"
done

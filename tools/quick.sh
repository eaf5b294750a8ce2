#!/bin/bash
# Quick GPU iteration: full -m gpu suite, then bench lines (default C2 and C4;
# CONFIGS="C1 C2 C4 C5obs" to choose; C5obs = C5's observed pattern alone).
#   gpurun --timeout 1200 -- 'bash tools/quick.sh TAG [pytest args]'
tag=${1:-q}; shift
out=gpurun_out; mkdir -p $out
if [[ -z $NO_TESTS ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q -rs "$@" > $out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> $out/pytest_$tag.log
  tail -3 $out/pytest_$tag.log
fi
for c in ${CONFIGS:-C2 C4}; do
  extra=""; cc=$c
  if [[ $c == C5obs ]]; then cc=C5; extra="--sims 0"; fi
  timeout 300 python bench.py --config $cc $extra --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$tag.json 2> $out/bench_${c}_$tag.err
  python -c "import json;d=json.load(open('$out/bench_${c}_$tag.json'));r=d['roofline'];print('$c', round(d['ms_per_step'],3), 'ms; dev', round(d['device_ms_per_step'],3), 'pair', round(r['kernel_ms_per_step'],3), 'grid', round(r['grid_build']['ms_per_step'],3), 'frac', round(r['grid_build']['frac'],3))"
done

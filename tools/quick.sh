#!/bin/bash
# Quick GPU iteration: full -m gpu suite, then C2 and C4 bench lines.
#   gpurun --timeout 1200 -- 'bash tools/quick.sh TAG [pytest args]'
tag=${1:-q}; shift
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -rs "$@" > $out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> $out/pytest_$tag.log
tail -3 $out/pytest_$tag.log
for c in C2 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$tag.json 2> $out/bench_${c}_$tag.err
  python -c "import json;d=json.load(open('$out/bench_${c}_$tag.json'));print('$c', round(d['ms_per_step'],2), 'ms', d['roofline']['kernel_ms_per_step'])"
done

#!/bin/bash
# ncu on the non-pair kernels: K1 grid build (key / place / gather / scan) on C4
# and on C5's observed pattern (full sets), and C1's launch list (small-job latency).
#   gpurun --timeout 1800 -- 'bash tools/ncu_small.sh TAG'
tag=${1:-k1}
out=gpurun_out; mkdir -p $out
k1='regex:key_kernel|place_kernel|gather_kernel|scan_kernel|csr_gen_kernel|csr_finish_kernel'
timeout 600 python bench.py --config C5 --sims 0 --steps 1 --warmup 1 --no-cpu-baseline > $out/b_c5obs_$tag.json 2>&1
timeout 600 ncu --set full --clock-control none -k "$k1" -c 4 -o $out/k1_C5obs_$tag -f \
  python bench.py --config C5 --sims 0 --steps 1 --warmup 0 --no-cpu-baseline > $out/ncu_k1_C5obs_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none -k "$k1" -c 6 -o $out/k1_C4_$tag -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $out/ncu_k1_C4_$tag.log 2>&1
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > $out/b_c1_$tag.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_C1_$tag.csv python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline \
  > $out/ncu_c1_$tag.log 2>&1
echo done

#!/bin/bash
# One GPU-box session: parity tests, the default bench line, the other configs,
# the ncu launch list and full captures of the pair kernel.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag] [stages]'
# stages: any of t (tests) s (smoke) b (bench default C4 + reference arm) c (other
# configs) k (K1 on C5's observed pattern, permutation timing) p (polygons) l (launch
# list) f (ncu full: C4 and C2)
tag=${1:-r2}
stages=${2:-tbclf}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu_$tag.txt 2>&1
python -c "from paper_1912_04753_b200 import build; print(build.source_hash())" > $out/src_hash_$tag.txt
if [[ $stages == *t* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rs > $out/pytest_gpu_$tag.log 2>&1
  echo "pytest rc=$?" >> $out/pytest_gpu_$tag.log
fi
if [[ $stages == *s* ]]; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1
  echo "smoke rc=$?" >> $out/smoke_$tag.log
fi
if [[ $stages == *b* ]]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_$tag.json 2> $out/bench_$tag.err
  echo "bench rc=$?" >> $out/bench_$tag.err
  timeout 1200 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup ${REF_WARMUP:-1} > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
fi
if [[ $stages == *c* ]]; then
  for c in C1 C2 C3; do
    timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$tag.json 2> $out/bench_${c}_$tag.err
  done
  timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > $out/bench_C5_$tag.json 2> $out/bench_C5_$tag.err
fi
if [[ $stages == *k* ]]; then  # K1 grid build on C5's clustered observed pattern alone
  timeout 600 python bench.py --config C5 --sims 0 --steps 3 --warmup 2 --no-cpu-baseline > $out/bench_C5obs_$tag.json 2> $out/bench_C5obs_$tag.err
  timeout 600 python tools/perm_time.py 1000000 10 > $out/perm_par_$tag.json 2>&1
fi
if [[ $stages == *p* ]]; then
  for v in 128 512 2048; do
    timeout 600 python bench.py --config C2 --ring $v --steps 2 --warmup 2 --cpu-sample-frac 0.1 > $out/bench_ring${v}_$tag.json 2> $out/bench_ring${v}_$tag.err
  done
fi
if [[ $stages == *l* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $out/ncu_launch_$tag.log 2>&1
fi
if [[ $stages == *f* ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
    -o $out/pair_kernel_C4_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > $out/ncu_full_C4_$tag.log 2>&1
  echo "ncu rc=$?" >> $out/ncu_full_C4_$tag.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
    -o $out/pair_kernel_C2_$tag -f python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline \
    > $out/ncu_full_C2_$tag.log 2>&1
  echo "ncu rc=$?" >> $out/ncu_full_C2_$tag.log
fi
echo done

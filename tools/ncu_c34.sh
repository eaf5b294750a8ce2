out=gpurun_out; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 1 -c 1 -o $out/pair_kernel_C3 -f python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline > $out/ncu_C3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 1 -c 1 -o $out/pair_kernel_C4 -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline > $out/ncu_C4.log 2>&1
echo done

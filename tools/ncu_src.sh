# Source-counter capture of one pair-kernel launch:
#   bash tools/ncu_src.sh CFG TAG "EXTRA BENCH ARGS" [ENV=VALUE ...]
out=gpurun_out; mkdir -p $out
cfg=$1; tag=$2; extra=$3; shift 3
env "$@" timeout 1200 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section SpeedOfLight --clock-control none --import-source on \
  -k regex:pair_kernel -s 1 -c 1 -o $out/src_${cfg}_$tag -f python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline $extra > $out/ncu_src_${cfg}_$tag.log 2>&1
echo "ncu $cfg $tag rc=$?"

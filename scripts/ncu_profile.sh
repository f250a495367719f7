#!/bin/bash
# Run under gpurun: launch list + one `ncu --set full` capture of each attention kernel.
#   gpurun -- 'bash scripts/ncu_profile.sh <tag> [prefill_regex] [decode_regex]'
set -u
TAG=${1:-r01}
PRE=${2:-prefill}
DEC=${3:-decode_pair_kernel}
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
# 1) every launch with its device time (cold-cache, serialised: compare SHARES)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 --no-sweep --no-comparator --no-ablation > $OUT/${TAG}_launches_bench.log 2>&1
# 2) full sections of the dominant kernels (one launch each, after warm-up)
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$PRE -s 3 -c 1 \
  -o $OUT/${TAG}_prefill python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c4 --no-sweep --no-comparator --no-ablation > $OUT/${TAG}_prefill_ncu.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$DEC -s 3 -c 1 \
  -o $OUT/${TAG}_decode python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c4 --no-sweep --no-comparator --no-ablation > $OUT/${TAG}_decode_ncu.log 2>&1
ls -la $OUT

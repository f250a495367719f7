#!/bin/bash
# Experiment: time the prefill kernel with parts of its arithmetic removed (HACK_ABL=n).
for a in ${ABLS:-0 1 2 3 4}; do
  touch paper_2502_03589_b200/csrc/prefill_tc.cu
  HACK_EXTRA_NVCC_FLAGS="-DHACK_ABL=$a" python paper_2502_03589_b200/build.py > /dev/null 2>&1 || { echo "build $a failed"; continue; }
  echo "ABL=$a $(timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | grep -o '"achieved": [0-9.]*' | head -1)"
done
touch paper_2502_03589_b200/csrc/prefill_tc.cu

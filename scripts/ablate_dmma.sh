#!/bin/bash
# Experiment: decode_mma_kernel shape sweep on the C4 (G = 8) decode sub-benchmark.
#   CFGS="4,8,3 3,6,4" bash scripts/ablate_dmma.sh
for c in ${CFGS:-4,8,3}; do
  IFS=, read nw ns ct <<< "$c"
  touch paper_2502_03589_b200/csrc/decode_mma.cu
  HACK_EXTRA_NVCC_FLAGS="-DHACK_DMMA_NW=$nw -DHACK_DMMA_NSTG=$ns -DHACK_DMMA_CTAS=$ct" python paper_2502_03589_b200/build.py > /tmp/b.log 2>&1 || { echo "build $c failed"; tail -5 /tmp/b.log; continue; }
  echo "NW=$nw NSTG=$ns CTAS=$ct $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-comparator --no-sweep --no-ablation 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read())["c4"]["per_bits"]; print({b: round(v["decode_kv_gbs"]) for b, v in d.items()})')"
done
touch paper_2502_03589_b200/csrc/decode_mma.cu
python paper_2502_03589_b200/build.py > /dev/null 2>&1  # leave the default build in place

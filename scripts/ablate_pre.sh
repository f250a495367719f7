#!/bin/bash
# Experiment: prefill_tc compile-time variants: FLAGS="-DX=1|-DX=2" bash scripts/ablate_pre.sh
IFS='|' read -ra V <<< "${FLAGS:-}"
for f in "${V[@]}"; do
  touch paper_2502_03589_b200/csrc/prefill_tc.cu
  HACK_EXTRA_NVCC_FLAGS="$f" python paper_2502_03589_b200/build.py > /tmp/b.log 2>&1 || { echo "build '$f' failed"; tail -5 /tmp/b.log; continue; }
  echo "[$f] $(timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("kernel TOPS", round(d["roofline"]["achieved"],1), "step TOPS", round(d["value"],1))')"
done
touch paper_2502_03589_b200/csrc/prefill_tc.cu

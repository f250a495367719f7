#!/bin/bash
# prefill timing ablations (wrong results): HACK_ABL bit flags, one bench line each
for a in "$@"; do
  HACK_EXTRA_NVCC_FLAGS="-DHACK_ABL=$a" python paper_2502_03589_b200/build.py > /dev/null
  python bench.py --steps 10 --warmup 3 --no-sweep --no-c4 --no-comparator --no-ablation --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ABL=$a', round(l['roofline']['achieved'],1), 'TOPS kernel')"
done
python paper_2502_03589_b200/build.py > /dev/null

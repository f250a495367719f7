#!/bin/bash
# A/B timing of two prefill_tc.cu variants on one box: ab.sh other.cu
b() { python bench.py --steps 10 --warmup 3 --no-sweep --no-c4 --no-comparator --no-ablation --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['roofline']['achieved'],1))"; }
cp paper_2502_03589_b200/csrc/prefill_tc.cu /tmp/cur.cu
b cur; cp $1 paper_2502_03589_b200/csrc/prefill_tc.cu; python paper_2502_03589_b200/build.py > /dev/null; b other
cp /tmp/cur.cu paper_2502_03589_b200/csrc/prefill_tc.cu; python paper_2502_03589_b200/build.py > /dev/null; b cur

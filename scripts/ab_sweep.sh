#!/bin/bash
# A/B of libhack builds on the Pi x bits sweep and C4 (decode_mma paths):
#   bash scripts/ab_sweep.sh name1 name2 ...   (abtest/libhack_<name>.so)
cd $GRAFT_REPO_ROOT
cp paper_2502_03589_b200/libhack.so /tmp/libhack_orig.so
for r in 1 2; do for v in "$@"; do
  cp abtest/libhack_$v.so paper_2502_03589_b200/libhack.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-comparator --no-ablation --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); c4=l.get('c4') or {}
print('== $v', 'sweep dec GB/s', [(p['Pi'], p['bits'], round(p['decode_kv_gbs'])) for p in l['pi_bits_sweep']['points']],
      '| c4', {k: round(v['decode_kv_gbs']) for k, v in (c4.get('per_bits') or {}).items()})"
done; done
cp /tmp/libhack_orig.so paper_2502_03589_b200/libhack.so

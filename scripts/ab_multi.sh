#!/bin/bash
# A/B several builds of libhack.so on one box, two rounds, decode + prefill bench lines:
#   bash scripts/ab_multi.sh name1 name2 ...   (abtest/libhack_<name>.so)
cd $GRAFT_REPO_ROOT
cp paper_2502_03589_b200/libhack.so /tmp/libhack_orig.so
for r in 1 2; do for v in "$@"; do
  cp abtest/libhack_$v.so paper_2502_03589_b200/libhack.so
  timeout 150 python bench.py --steps 20 --warmup 3 --no-sweep --no-comparator --no-ablation --no-cpu-baseline ${AB_ARGS} 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); d=l['decode']; c4=l.get('c4') or {}
print('== $v', 'pre %.1f' % l['roofline']['achieved'], '| dec attn_ms %.4f GB/s %.0f step_ms %.4f' % (d['attn_ms'], d['kv_gbs'], d['ms_per_step']),
      '| c4', {k: (round(v['prefill_tops']), round(v['decode_kv_gbs'])) for k, v in (c4.get('per_bits') or {}).items()})"
  if [ -n "$SHARD" ]; then python scripts/dec_shard_probe.py 8 2>&1 | tail -1; fi
done; done
cp /tmp/libhack_orig.so paper_2502_03589_b200/libhack.so

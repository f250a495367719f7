cd $GRAFT_REPO_ROOT
for r in 1 2; do for f in 0 1; do
  HACK_DECODE_FUSED=$f timeout 150 python bench.py --steps 20 --warmup 3 --no-sweep --no-comparator --no-ablation --no-cpu-baseline --no-c4 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); d=l['decode']
print('fused=$f', 'attn_ms %.4f step_ms %.4f GB/s %.0f' % (d['attn_ms'], d['ms_per_step'], d['kv_gbs']))"
done; done
for f in 0 1; do HACK_DECODE_FUSED=$f python scripts/dec_shard_probe.py 8 2>&1 | tail -1; done

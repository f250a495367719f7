#!/bin/bash
# decode iteration: decode tests (optional), a short bench line, the N = 8 shard probe
# usage (under gpurun): bash scripts/dec_quick.sh [pytest -k expr]
cd $GRAFT_REPO_ROOT
if [ -n "$1" ]; then timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$1" 2>&1 | tail -3; fi
python bench.py --steps 10 --warmup 3 --no-sweep --no-c4 --no-comparator --no-ablation --no-cpu-baseline > gpurun_out/b_dq.json 2>gpurun_out/b_dq.err
python - <<'PY'
import json
l = json.loads(open("gpurun_out/b_dq.json").read().strip().splitlines()[-1]); d = l["decode"]
print("prefill step %.1f kernel %.1f | decode attn ms %.4f GB/s %.0f step ms %.4f" % (
    l["value"], l["roofline"]["achieved"], d["attn_ms"], d["kv_gbs"], d["ms_per_step"]))
PY
for n in 1 2 4 8; do python scripts/dec_shard_probe.py $n; done; PROBE_SEPARATE=1 python scripts/dec_shard_probe.py 8

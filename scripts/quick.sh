#!/bin/bash
# quick GPU iteration: prefill/decode parity subset + a short bench line (no sweeps)
# usage: scripts/quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-"prefill or decode or c4"}
python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$K" > gpurun_out/t_$TAG.log 2>&1; tail -3 gpurun_out/t_$TAG.log
python bench.py --steps 10 --warmup 3 --no-sweep --no-c4 --no-comparator --no-ablation --no-cpu-baseline > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
python - <<PY
import json
l = json.loads(open("gpurun_out/b_$TAG.json").read().strip().splitlines()[-1])
d = l["decode"]
print("prefill step TOPS %.1f  kernel %.1f  ms %.4f | decode attn ms %.4f  KV GB/s %.0f  step ms %.4f" % (
    l["value"], l["roofline"]["achieved"], l["roofline"]["ms_per_launch"], d["attn_ms"], d["kv_gbs"], d["ms_per_step"]))
PY

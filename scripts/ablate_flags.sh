#!/bin/bash
# Experiment: rebuild with each extra nvcc flag set and print C3 decode GB/s + prefill TOPS.
#   FLAGS="-DHACK_DEC_PF=0|-DHACK_DEC_PF=8" bash scripts/ablate_flags.sh
IFS='|' read -ra SETS <<< "${FLAGS}"
for f in "${SETS[@]}"; do
  touch paper_2502_03589_b200/csrc/*.cu
  HACK_EXTRA_NVCC_FLAGS="$f" python paper_2502_03589_b200/build.py > /tmp/b.log 2>&1 || { echo "build [$f] failed"; tail -5 /tmp/b.log; continue; }
  echo "[$f] $(timeout 180 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-comparator --no-sweep ${BENCH_ARGS} 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); x=d["decode"]; c=d.get("c4") or {}; print("prefill", round(d["value"],1), "| C3 GB/s", round(x["kv_gbs"],1), "attn_ms", round(x["attn_ms"],4), "step_ms", round(x["ms_per_step"],4), "| C4", {k: round(v["decode_kv_gbs"],1) for k, v in (c.get("per_bits") or {}).items()})')"
done
touch paper_2502_03589_b200/csrc/*.cu
python paper_2502_03589_b200/build.py > /dev/null 2>&1  # leave the default build in place

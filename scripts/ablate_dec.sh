#!/bin/bash
# Experiment: decode_pair kernel shape sweep (compute warps / ring slots / CTAs per SM).
#   CFGS="4,12,3 8,18,2" bash scripts/ablate_dec.sh
for c in ${CFGS:-4,12,3,0}; do
  IFS=, read nw ns ct abl <<< "$c"
  abl=${abl:-0}
  touch paper_2502_03589_b200/csrc/decode_pair.cu
  HACK_EXTRA_NVCC_FLAGS="-DHACK_DEC_NW=$nw -DHACK_DEC_NSTG=$ns -DHACK_DEC_CTAS=$ct -DHACK_ABL=$abl" python paper_2502_03589_b200/build.py > /tmp/b.log 2>&1 || { echo "build $c failed"; tail -5 /tmp/b.log; continue; }
  echo "NW=$nw NSTG=$ns CTAS=$ct ABL=$abl $(timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c4 --no-sweep --no-ablation --no-comparator 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["decode"]["kv_gbs"],1), round(d["decode"]["attn_ms"],4))')"
done
touch paper_2502_03589_b200/csrc/decode_pair.cu
python paper_2502_03589_b200/build.py > /dev/null 2>&1  # leave the default build in place

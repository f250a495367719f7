#!/bin/bash
# A/B two builds of libhack.so on one box: bash scripts/ab_so.sh <cmd> (abtest/libhack_{head,new}.so)
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in head new; do
  cp abtest/libhack_$v.so paper_2502_03589_b200/libhack.so
  echo "== $v: $(eval "$1" 2>&1 | tail -1)"
done; done

cd $GRAFT_REPO_ROOT
for f in "" "-DHACK_DEC_STREAM" "-DHACK_DEC_STREAM -DHACK_DEC_NSTG=12 -DHACK_DEC_CTAS=3" "-DHACK_DEC_STREAM -DHACK_DEC_NSTG=6"; do
  touch paper_2502_03589_b200/csrc/decode_pair.cu
  HACK_EXTRA_NVCC_FLAGS="$f" python paper_2502_03589_b200/build.py > /tmp/b.log 2>&1 || { echo "build failed $f"; continue; }
  echo "[$f] $(PROBE_SEPARATE=1 python scripts/dec_shard_probe.py 1)"
done
touch paper_2502_03589_b200/csrc/decode_pair.cu; python paper_2502_03589_b200/build.py > /dev/null 2>&1

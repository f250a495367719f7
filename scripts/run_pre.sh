cd $GRAFT_REPO_ROOT
if [ "${TESTS:-1}" = 1 ]; then
timeout 900 python -m pytest tests/test_gpu_prefill.py -x -q > gpurun_out/pre_tests.log 2>&1; echo EXIT $? >> gpurun_out/pre_tests.log
tail -3 gpurun_out/pre_tests.log
fi
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_pre.json 2> gpurun_out/bench_pre.err
python - <<'PY'
import json, os
d=json.loads(open('gpurun_out/bench_pre.json').read().strip().splitlines()[-1])
print('prefill step TOPS', round(d['value'],1), 'kernel TOPS', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],4), 'ms', round(d['roofline']['ms_per_launch'],4), 'decode GB/s', round(d['decode']['kv_gbs'],1))
PY
if [ "${NCU:-0}" = 1 ]; then
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 \
  -o gpurun_out/pre_tc -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/pre_ncu.log 2>&1
tail -1 gpurun_out/pre_ncu.log
fi

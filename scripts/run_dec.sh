cd $GRAFT_REPO_ROOT
if [ "${TESTS:-1}" = 1 ]; then
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kv_transfer.py -x -q > gpurun_out/dec_tests.log 2>&1; echo EXIT $? >> gpurun_out/dec_tests.log
tail -3 gpurun_out/dec_tests.log
fi
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_dec.json 2> gpurun_out/bench_dec.err
python - <<'PY'
import json, os
d=json.loads(open('gpurun_out/bench_dec.json').read().strip().splitlines()[-1])
x=d['decode']
print('prefill', round(d['value'],1), 'kernel', round(d['roofline']['achieved'],1), '| decode GB/s', round(x['kv_gbs'],1), 'frac', round(x['roofline']['frac'],3), 'attn_ms', round(x['attn_ms'],4), 'step_ms', round(x['ms_per_step'],4))
PY
if [ "${NCU:-0}" = 1 ]; then
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-decode_pair_kernel} -s 3 -c 1 \
  -o gpurun_out/dec_pair -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/dec_ncu.log 2>&1
tail -1 gpurun_out/dec_ncu.log
fi

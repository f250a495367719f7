TAG=${1:-r04}
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_full.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests_full.log
tail -3 gpurun_out/gpu_tests_full.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
bash scripts/ncu_profile.sh ${TAG} > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu exit $?"
timeout 900 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"prefill_tc|decode_pair_kernel" -s 6 -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c4 --no-sweep --no-comparator --no-ablation > gpurun_out/traffic_${TAG}.csv 2>&1; echo "traffic exit $?"

#!/bin/bash
# Run under gpurun: compute-sanitizer (memcheck, racecheck, synccheck) over smoke() and a few
# small GPU tests that cover the clustered append, the no-RQE append, the paired / G=8
# decode kernels (fused step, in-kernel merge), prefill at Pi = 32 / 128 and P-SR, and the
# KV pack/unpack.  Logs -> gpurun_out/san_<tool>.log
OUT=gpurun_out
mkdir -p $OUT
SAN=/usr/local/cuda/bin/compute-sanitizer
TESTS="tests/test_gpu_rqe_ablation.py::test_no_rqe_requantizes_partial_block[2] tests/test_gpu_decode.py::test_decode_paired_kernel_edges tests/test_gpu_decode.py::test_decode_group8_paired_kernel[8-auto] tests/test_gpu_kv_transfer.py::test_pack_unpack_round_trip_and_decode_equivalence tests/test_gpu_decode.py::test_decode_partition_and_bits tests/test_gpu_kv_transfer.py::test_kv_pull_fused_transfer tests/test_gpu_kv_transfer.py::test_layer_pipelined_nccl_self_loop tests/test_gpu_decode.py::test_fused_decode_step_equals_separate[8-1] tests/test_gpu_decode.py::test_fused_decode_step_equals_separate[16-0] tests/test_gpu_decode.py::test_decode_workspace_reuse_merge_counters[8-1] tests/test_gpu_prefill.py::test_prefill_partition_and_bits[32-2] tests/test_gpu_prefill.py::test_prefill_partition_and_bits[128-4] tests/test_gpu_prefill.py::test_prefill_p_stochastic_rounding[300-4-2-2-64] tests/test_gpu_prefill.py::test_prefill_host_position_streamed_equals_device_call[1000--3-37-64-2]"
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  {
    timeout 600 $SAN --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()"
    echo "smoke exit $?"
    timeout 900 $SAN --tool $tool --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider $TESTS
    echo "tests exit $?"
  } > $OUT/san_$tool.log 2>&1
  grep -E "ERROR SUMMARY|exit|passed|failed" $OUT/san_$tool.log | tail -6
done

#!/bin/bash
set -u
mkdir -p gpurun_out/tcb
python scripts/tc_bench.py > gpurun_out/tcb/normal.txt 2>&1
MQGNN_LIB=$PWD/paper_2601_04707_b200/libmqgnn_trace.so python scripts/tc_bench.py > gpurun_out/tcb/trace.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fused.py tests/test_gpu_epoch.py -x -q > gpurun_out/tcb/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/tcb/pytest.log
cat gpurun_out/tcb/normal.txt; grep -A6 "FWD  M=   2604" gpurun_out/tcb/trace.txt; tail -n 3 gpurun_out/tcb/pytest.log

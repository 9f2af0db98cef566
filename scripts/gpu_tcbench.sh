#!/bin/bash
# tcgen05 GEMM micro-benchmark, normal + trace builds.
set -u
mkdir -p gpurun_out/tcb
python scripts/tc_bench.py > gpurun_out/tcb/normal.txt 2>&1
MQGNN_LIB=$PWD/paper_2601_04707_b200/libmqgnn_trace.so python scripts/tc_bench.py > gpurun_out/tcb/trace.txt 2>&1
cat gpurun_out/tcb/normal.txt gpurun_out/tcb/trace.txt

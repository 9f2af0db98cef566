#!/bin/bash
# TMA GEMM (v2) bring-up: tcgen05 parity tests, then the micro-benchmark of
# both kernel versions.  Usage: gpurun -- 'bash scripts/gpu_tc2.sh TAG'
set -u
TAG=${1:-tc2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > $OUT/pytest_tc.log 2>&1; echo "exit $?" >> $OUT/pytest_tc.log
tail -n 30 $OUT/pytest_tc.log
timeout 300 python scripts/tc_bench.py > $OUT/bench.txt 2>&1; echo "exit $?" >> $OUT/bench.txt
cat $OUT/bench.txt

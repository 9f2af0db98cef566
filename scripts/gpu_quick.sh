#!/bin/bash
# Quick GPU check: selected GPU tests + default bench (per-op table).
# Usage: gpurun --timeout 1200 -- 'bash scripts/gpu_quick.sh TAG "pytest selection" ["bench args"]'
set -u
TAG=$1; SEL=${2:-tests}; BARGS=${3:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest $SEL -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
MQ_BENCH_KERNELS=1 timeout 600 python bench.py --no-cpu-baseline $BARGS > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -n 3 $OUT/pytest_gpu.log; tail -n 2 $OUT/bench.err
python scripts/show_bench.py $OUT/bench.jsonl 2>&1 | head -20

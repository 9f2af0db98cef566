#!/bin/bash
# Iteration pass: selected GPU tests, default bench (per-op table), ncu --set
# full of kernels matching REGEX (exported to CSV).
# Usage: gpurun --timeout 1800 -- 'bash scripts/gpu_iter.sh TAG "pytest selection" REGEX COUNT'
set -u
TAG=$1; SEL=${2:-tests}; RE=${3:-}; CNT=${4:-4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest $SEL -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
MQ_BENCH_KERNELS=1 timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ -n "$RE" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s ${SKIP:-40} -c $CNT \
    -o $OUT/prof python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 \
    --e2e-steps 3 > $OUT/ncu.log 2>&1; echo "ncu exit $?" >> $OUT/ncu.log
  bash scripts/ncu_export.sh $OUT > /dev/null 2>&1
fi
tail -n 3 $OUT/pytest_gpu.log; tail -n 2 $OUT/bench.err
python scripts/show_bench.py $OUT/bench.jsonl 2>&1 | head -20

#!/bin/bash
# A/B of environment settings on the default bench (per-op table kept).
# Usage: gpurun -- 'bash scripts/gpu_ab_env.sh TAG "pytest selection" "ENV=a" "ENV=b" ...'
set -u
TAG=$1; SEL=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$SEL" ]; then
  timeout 900 python -m pytest $SEL -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
  tail -n 2 $OUT/pytest_gpu.log
fi
i=0
for E in "$@"; do
  i=$((i+1))
  env $E MQ_BENCH_KERNELS=1 timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$i.jsonl 2> $OUT/bench_$i.err
  echo "== $E"; python scripts/show_bench.py $OUT/bench_$i.jsonl 2>&1 | head -1
done

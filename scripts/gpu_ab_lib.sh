#!/bin/bash
# A/B of library builds on the default bench (each variant a separate .so,
# selected with MQGNN_LIB; per-op table kept).
# Usage: gpurun -- 'bash scripts/gpu_ab_lib.sh TAG "pytest selection" lib_a.so lib_b.so ...'
set -u
TAG=$1; SEL=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$SEL" ]; then
  for L in "$@"; do
    MQGNN_LIB=$L timeout 900 python -m pytest $SEL -m gpu -x -q > $OUT/pytest_$(basename $L).log 2>&1
    echo "pytest $L exit $?"; tail -n 1 $OUT/pytest_$(basename $L).log
  done
fi
for rep in 1 2; do
  for L in "$@"; do
    b=$(basename $L .so)
    MQGNN_LIB=$L MQ_BENCH_KERNELS=1 timeout 600 python bench.py --no-cpu-baseline --steps 1500 --e2e-steps 600 \
      > $OUT/bench_${b}_$rep.jsonl 2> $OUT/bench_${b}_$rep.err
    echo "== $L rep $rep"; python scripts/show_bench.py $OUT/bench_${b}_$rep.jsonl 2>&1 | grep -E "seeds/s|aggregate|optimizer"
  done
done

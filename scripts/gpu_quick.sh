#!/bin/bash
# Quick GPU pass: selected tests + a short bench (+ optional launch list).
# Usage: gpurun -- 'bash scripts/gpu_quick.sh TAG "pytest args" [ncu]'
set -u
TAG=${1:-quick}
TESTS=${2:-tests -m gpu -x -q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "$TESTS" != "none" ]; then
  timeout 900 python -m pytest $TESTS > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
fi
MQ_BENCH_KERNELS=1 timeout 600 python bench.py --no-cpu-baseline --steps 600 > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ "${3:-}" = "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 30 --warmup 3 --no-cpu-baseline --profile-steps 0 --e2e-steps 10 > $OUT/ncu_bench.log 2>&1
  echo "ncu exit $?" >> $OUT/ncu_bench.log
fi
for f in $OUT/pytest.log $OUT/bench.err; do [ -f $f ] && { echo "== $f"; tail -n 25 $f; }; done
head -c 1500 $OUT/bench.jsonl

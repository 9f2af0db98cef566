#!/bin/bash
# GPU tests + reddit/products bench lines (+ per-kernel table).  Usage: gpurun -- 'bash scripts/gpu_check.sh TAG [pytest-args]'
set -u
TAG=${1:-chk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest ${2:-tests -m gpu -x -q} > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
MQ_BENCH_KERNELS=1 timeout 400 python bench.py --no-cpu-baseline > $OUT/reddit.jsonl 2> $OUT/reddit.err
MQ_BENCH_KERNELS=1 timeout 600 python bench.py --shape products --steps 300 --no-cpu-baseline > $OUT/products.jsonl 2> $OUT/products.err
tail -n 3 $OUT/pytest.log
for f in $OUT/reddit.jsonl $OUT/products.jsonl; do python scripts/show_bench.py $f; done
tail -n 3 $OUT/*.err

#!/bin/bash
# GPU pass for the per-epoch functions + a default bench line.
# Usage: gpurun -- 'bash scripts/gpu_epoch.sh TAG'
set -u
TAG=${1:-ep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_epoch.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python scripts/epoch_timing.py --shape reddit > $OUT/reddit.json 2> $OUT/reddit.err
timeout 400 python scripts/epoch_timing.py --shape products > $OUT/products.json 2> $OUT/products.err
MQ_BENCH_KERNELS=1 timeout 600 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -n 5 $OUT/pytest.log; cat $OUT/reddit.json $OUT/products.json; tail -n 3 $OUT/reddit.err $OUT/products.err $OUT/bench.err

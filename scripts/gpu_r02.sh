#!/bin/bash
# Round-2 GPU pass: full GPU suite, smoke, Reddit bench, 2-rank functional runs
# (ranks share the one GPU: gloo plumbing, peer-memory data path).
# Usage: gpurun --timeout 3000 -- 'bash scripts/gpu_r02.sh TAG'
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
MQ_BENCH_KERNELS=1 timeout 600 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
MQ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --shape products --steps 200 --no-cpu-baseline --feature-placement sharded > $OUT/products_2rank_sharded.jsonl 2> $OUT/products_2rank.err; echo "exit $?" >> $OUT/products_2rank.err
for f in $OUT/*.log $OUT/*.err; do echo "== $f"; tail -n 3 $f; done

#!/bin/bash
# Closing GPU pass: full GPU suite, smoke, the default bench, products /
# papers / reference lines, ncu launch list of a short default bench.
# Usage: gpurun --timeout 3600 -- 'bash scripts/gpu_final.sh TAG'
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
MQ_BENCH_KERNELS=1 timeout 600 python bench.py > $OUT/reddit.jsonl 2> $OUT/reddit.err; echo "exit $?" >> $OUT/reddit.err
timeout 600 python bench.py --impl reference > $OUT/reference.jsonl 2> $OUT/reference.err; echo "exit $?" >> $OUT/reference.err
MQ_BENCH_KERNELS=1 timeout 900 python bench.py --shape products --steps 600 --no-cpu-baseline > $OUT/products.jsonl 2> $OUT/products.err; echo "exit $?" >> $OUT/products.err
MQ_BENCH_KERNELS=1 timeout 1500 python bench.py --shape papers --steps 300 --warmup 5 --e2e-steps 100 --profile-steps 5 > $OUT/papers.jsonl 2> $OUT/papers.err; echo "exit $?" >> $OUT/papers.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline --profile-steps 2 --e2e-steps 10 > $OUT/ncu_bench.log 2>&1; echo "ncu exit $?" >> $OUT/ncu_bench.log
for f in $OUT/*.log $OUT/*.err; do echo "== $f"; tail -n 2 $f; done
for f in $OUT/*.jsonl; do python scripts/show_bench.py $f 2>&1 | head -1; done

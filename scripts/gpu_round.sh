#!/bin/bash
# One GPU box pass: build check, parity tests, smoke, bench, ncu launch list.
# Usage (from this container): gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh TAG'
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
MQ_BENCH_KERNELS=1 timeout 600 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline --profile-steps 2 --e2e-steps 10 > $OUT/ncu_bench.log 2>&1; echo "ncu exit $?" >> $OUT/ncu_bench.log
for f in $OUT/*.log $OUT/bench.err; do echo "== $f"; tail -n 3 $f; done

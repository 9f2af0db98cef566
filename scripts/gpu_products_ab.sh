#!/bin/bash
# products-shape bench under several environments (crash / perf A/B)
# Usage: gpurun -- 'bash scripts/gpu_products_ab.sh TAG STEPS "ENV=a" "ENV=b" ...'
set -u
TAG=$1; STEPS=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
i=0
for E in "$@"; do
  i=$((i+1))
  env $E timeout 900 python bench.py --shape products --no-cpu-baseline --steps $STEPS --profile-steps 1 --e2e-steps 50 > $OUT/p_$i.jsonl 2> $OUT/p_$i.err
  echo "== $E exit $?"; python scripts/show_bench.py $OUT/p_$i.jsonl 2>&1 | head -1; grep -m1 "Error" $OUT/p_$i.err
done

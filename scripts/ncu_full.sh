#!/bin/bash
# ncu --set full capture of selected kernels of a short bench run (1 GPU).
# Usage: gpurun -- 'bash scripts/ncu_full.sh TAG "regex" COUNT ["extra bench args"]'
set -u
TAG=$1; RE=$2; CNT=${3:-6}; EXTRA=${4:-}
mkdir -p gpurun_out/$TAG
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s ${SKIP:-40} -c $CNT \
  -o gpurun_out/$TAG/prof python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 \
  --e2e-steps 3 $EXTRA > gpurun_out/$TAG/ncu.log 2>&1
echo "ncu exit $?"; tail -5 gpurun_out/$TAG/ncu.log

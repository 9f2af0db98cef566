#!/bin/bash
# Run each GPU test file under its own short timeout (a hung kernel costs
# one file, not the whole call).  Usage: gpurun -- 'bash scripts/gpu_files.sh TAG [secs]'
set -u
TAG=${1:-files}
T=${2:-150}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for f in tests/test_gpu_tc.py tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_runtime.py tests/test_gpu_epoch.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py; do
  n=$(basename $f .py)
  timeout $T python -m pytest $f -x -q --timeout 60 > $OUT/$n.log 2>&1
  echo "$n exit $? :: $(tail -n 1 $OUT/$n.log)"
done

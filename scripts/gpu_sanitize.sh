#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the kernel-level GPU
# tests: per-op kernels, the production prep pass, the fused step, the peer
# exchange kernels.  Logs go to gpurun_out/TAG/; summaries are copied into
# profiles/ by hand.  Usage: gpurun --timeout 3600 -- 'bash scripts/gpu_sanitize.sh TAG'
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL=${SEL:-"tests/test_gpu_parity.py tests/test_gpu_prep.py tests/test_gpu_fused.py::test_fused_three_layer_g2 tests/test_gpu_fused.py::test_group_graphs_match_window_graphs tests/test_gpu_peer.py::test_publish_apply_equal_accumulator_and_optimizer tests/test_gpu_peer.py::test_lagged_apply_holds_back_one_window tests/test_gpu_layerwise.py tests/test_gpu_tc.py::test_deferred_partials_repeated"}
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 9 \
    python -m pytest $SEL -x -q -p no:cacheprovider > $OUT/$tool.log 2>&1
  echo "$tool exit $?" >> $OUT/$tool.log
  tail -n 4 $OUT/$tool.log
done

#!/bin/bash
# GPU tests + bench A/B variants.  Usage: gpurun -- 'bash scripts/gpu_ab.sh TAG "variant args;..."'
set -u
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
IFS=';' read -ra VARS <<< "${2:-}"
i=0
for v in "" "${VARS[@]}"; do
  timeout 300 python bench.py --no-cpu-baseline --profile-steps 0 --e2e-steps 150 $v > $OUT/bench_$i.jsonl 2> $OUT/bench_$i.err
  echo "[$i] $v :: $(python -c "import json,sys; b=json.loads(open('$OUT/bench_$i.jsonl').readline()); print(round(b['value']/1e6,3),'M/s', round(b['ms_per_step']*1e3,2),'us/step e2e', round(b['e2e']['value']/1e6,3) if b.get('e2e') else None)" 2>&1)" >> $OUT/summary.txt
  i=$((i+1))
done
tail -n 3 $OUT/pytest.log; cat $OUT/summary.txt

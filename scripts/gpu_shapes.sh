#!/bin/bash
# Bench lines on the other BASELINE shapes: products (cfg3) and the cache /
# host-miss sweep (cfg4).  Usage: gpurun -- 'bash scripts/gpu_shapes.sh TAG'
set -u
TAG=${1:-shapes}
OUT=gpurun_out/$TAG
mkdir -p $OUT
MQ_BENCH_KERNELS=1 timeout 900 python bench.py --shape products --steps 600 > $OUT/products.jsonl 2> $OUT/products.err
for f in 0.001 0.01 0.1; do
  for p in hbm host; do
    timeout 600 python bench.py --shape products --steps 300 --no-cpu-baseline --profile-steps 5 \
      --e2e-steps 50 --cache-fraction $f --feature-placement $p > $OUT/sweep_${f}_${p}.jsonl 2> $OUT/sweep_${f}_${p}.err
  done
done
for f in $OUT/*.jsonl; do echo "$f :: $(python -c "import json; b=json.loads(open('$f').readline()); print(round(b['value']/1e6,3),'M/s', round(b['ms_per_step']*1e3,1),'us/step', 'e2e', round(b['e2e']['value']/1e6,3) if b.get('e2e') else None, 'hits', (b.get('cache') or {}).get('hit_rate'), 'host_link', {k: (b['host_link'] or {}).get(k) for k in ('achieved','peak','frac')} if b.get('host_link') else None)" 2>&1 | tail -1)"; done
tail -n 3 $OUT/*.err

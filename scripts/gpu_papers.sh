#!/bin/bash
# papers100M-shaped bench line (BASELINE configs[4]) on one B200.
set -u
mkdir -p gpurun_out/papers
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/papers/smi.txt
MQ_BENCH_KERNELS=1 timeout 1500 python bench.py --shape papers --steps 300 --warmup 5 --e2e-steps 100 --profile-steps 5 > gpurun_out/papers/bench.jsonl 2> gpurun_out/papers/bench.err
echo "exit $?" >> gpurun_out/papers/bench.err
python scripts/show_bench.py gpurun_out/papers/bench.jsonl; tail -n 5 gpurun_out/papers/bench.err
python -c "import json; b=json.loads(open('gpurun_out/papers/bench.jsonl').readline()); print(json.dumps({k: b.get(k) for k in ('setup','per_epoch','cache','epoch_ms','windows_per_epoch')}))"

bash scripts/gpu_quick.sh r03c "tests/test_gpu_prep.py tests/test_gpu_fused.py tests/test_gpu_runtime.py tests/test_gpu_fullsize.py"
MQ_BENCH_KERNELS=1 timeout 600 python bench.py --no-cpu-baseline --shape products > gpurun_out/r03c/bench_products.jsonl 2> gpurun_out/r03c/bench_products.err
python scripts/show_bench.py gpurun_out/r03c/bench_products.jsonl 2>&1 | head -20

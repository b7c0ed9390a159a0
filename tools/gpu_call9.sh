# run-cache change: e2e / multi / paged parity, then the bench line (e2e vs device)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_paged.py tests/test_gpu_fp32.py tests/test_gpu_t5.py -q > gpurun_out/pytest_cache.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_cache.log
timeout 1500 python bench.py > gpurun_out/bench_cache.json 2> gpurun_out/bench_cache.err; echo "bench rc $?"

# multi-GPU executors after the table-ring cache: multi + paged + T5 suites
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_paged.py tests/test_gpu_t5.py tests/test_gpu_fullsize.py -q > gpurun_out/pytest_multi_cache.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_multi_cache.log

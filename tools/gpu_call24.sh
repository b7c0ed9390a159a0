mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_paged.py tests/test_gpu_t5.py -q > gpurun_out/pytest24.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest24.log

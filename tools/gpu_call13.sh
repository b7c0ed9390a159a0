# final code: kernel + T5 suites (FMHA smem-P default, race/repeatability test)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_t5.py -q > gpurun_out/pytest_k13.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_k13.log

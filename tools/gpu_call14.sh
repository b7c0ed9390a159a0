mkdir -p gpurun_out
timeout 300 python tools/fmha_pt_check.py > gpurun_out/fmha_pt_check.log 2>&1; echo "check rc $?"
cat gpurun_out/fmha_pt_check.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_t5.py -q > gpurun_out/pytest_k14.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_k14.log

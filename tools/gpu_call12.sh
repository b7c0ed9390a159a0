# FMHA P-in-TMEM (WAR wait before S overwrites P): parity first, then the A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_t5.py tests/test_gpu_e2e.py tests/test_gpu_paged.py -x -q > gpurun_out/pytest_pt.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_pt.log
timeout 300 python tools/probe_kernels.py pmix_pt > gpurun_out/fmha_pt.log 2>&1; echo "A/B rc $?"
cat gpurun_out/fmha_pt.log

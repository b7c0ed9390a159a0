# FMHA P in TMEM as the default: kernel / T5 / e2e / paged / full-width suites, A/B, and the OPT-13B phase A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_t5.py tests/test_gpu_e2e.py tests/test_gpu_paged.py tests/test_gpu_fullsize.py tests/test_gpu_fp32.py -q > gpurun_out/pytest_pt_default.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_pt_default.log
timeout 300 python tools/probe_kernels.py pmix_pt > gpurun_out/fmha_pt.log 2>&1; echo "A/B rc $?"
cat gpurun_out/fmha_pt.log
timeout 300 python tools/fmha_pt_check.py > gpurun_out/fmha_pt_check.log 2>&1; cat gpurun_out/fmha_pt_check.log

# after linking torch's NCCL: smoke, multi (NCCL loopback), e2e, paged suites
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1; echo "smoke rc $?"; cat gpurun_out/smoke21.log
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_e2e.py tests/test_gpu_paged.py -q > gpurun_out/pytest21.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest21.log

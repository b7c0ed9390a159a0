mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -q > gpurun_out/pytest26.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest26.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

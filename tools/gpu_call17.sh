# final code: full GPU suite
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final2.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu_final2.log

# CTA-pair prefill GEMM: A/B + bitwise check vs the 1-CTA kernel, then the GEMM / e2e parity tests
mkdir -p gpurun_out
timeout 300 python tools/probe_kernels.py pgemm > gpurun_out/pair_ab.txt 2>&1; echo "probe rc $?"
cat gpurun_out/pair_ab.txt
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py tests/test_gpu_t5.py -m gpu -x -q > gpurun_out/pytest_pair.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_pair.log

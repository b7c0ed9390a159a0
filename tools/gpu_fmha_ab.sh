# FMHA A/B + parity: prefill attention probes (other builds vs this one),
# GPU kernel / T5 / e2e tests
mkdir -p gpurun_out
: > gpurun_out/fmha_ab.txt
for v in _p8; do
  if [ -f tools/$v/libexegpt.so ]; then
    echo "== $v" >> gpurun_out/fmha_ab.txt
    EXG_PROBE_LIB=$PWD/tools/$v/libexegpt.so timeout 300 python tools/probe_kernels.py pmix >> gpurun_out/fmha_ab.txt 2>&1
  fi
done
echo "== new" >> gpurun_out/fmha_ab.txt
timeout 300 python tools/probe_kernels.py pmix >> gpurun_out/fmha_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_t5.py tests/test_gpu_e2e.py -m gpu -x -q > gpurun_out/pytest_fmha.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_fmha.log
cat gpurun_out/fmha_ab.txt

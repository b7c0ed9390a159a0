# paged tests, FMHA prefetch A/B, decode GEMM timelines, config 3 fidelity, full GPU suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_paged.py -x -q > gpurun_out/pytest_paged.log 2>&1; echo "paged rc $?"
tail -3 gpurun_out/pytest_paged.log
timeout 300 python tools/probe_kernels.py pmix_pf > gpurun_out/fmha_pf.log 2>&1; echo "fmha A/B rc $?"
timeout 300 python tools/probe_timeline.py 64 20480 5120 > gpurun_out/tl_ffn1.log 2>&1; echo "tl ffn1 rc $?"
timeout 300 python tools/probe_timeline.py 83 15360 5120 > gpurun_out/tl_qkv.log 2>&1; echo "tl qkv rc $?"
timeout 1500 python tools/config3.py > gpurun_out/r2_config3.json 2> gpurun_out/config3.err; echo "config3 rc $?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc $?"
tail -4 gpurun_out/pytest_gpu_full.log

# final binary: full GPU suite, then the default bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final3.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu_final3.log
timeout 1500 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo "bench rc $?"

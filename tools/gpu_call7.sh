# paged multi-GPU tests (after the encoder-table fix), sanitizer incl. paged KV, configs 4/5 plans, second bench sample
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paged.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_paged_multi.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_paged_multi.log
timeout 1500 python tools/plan_configs.py > gpurun_out/r2_plans.json 2> gpurun_out/plans.err; echo "plans rc $?"
timeout 1500 python bench.py > gpurun_out/bench_sample2.json 2> gpurun_out/bench_sample2.err; echo "bench rc $?"

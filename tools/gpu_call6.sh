# configs 3 and 4 after the decode-context reading: T5 fidelity (1024 requests), OPT-66B slots vs pages
mkdir -p gpurun_out
timeout 1800 python tools/config3.py 1024 > gpurun_out/r2_config3_1024_ctx.json 2> gpurun_out/config3.err; echo "config3 rc $?"
timeout 1500 python bench.py --plan-dry-run --steps 3 --warmup 3 --requests 1024 > gpurun_out/c4_slots.json 2> gpurun_out/c4_slots.err; echo "c4 slots rc $?"
timeout 1500 python bench.py --plan-dry-run --kv-page 64 --steps 3 --warmup 3 --requests 1024 > gpurun_out/c4_paged.json 2> gpurun_out/c4_paged.err; echo "c4 paged rc $?"
timeout 1200 python -m pytest tests/test_gpu_paged.py tests/test_gpu_multi.py -q > gpurun_out/pytest_paged_multi.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_paged_multi.log

# paged KV (NEXT-2) verification + config-4 dry runs (slots vs pages) + config 3 (T5) fidelity
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_paged.py tests/test_gpu_kernels.py -k "paged" -x -q > gpurun_out/pytest_paged.log 2>&1; echo "paged tests rc $?"
tail -3 gpurun_out/pytest_paged.log
timeout 1500 python bench.py --plan-dry-run --steps 2 --warmup 1 --requests 1024 > gpurun_out/c4_slots.json 2> gpurun_out/c4_slots.err; echo "c4 slots rc $?"
timeout 1500 python bench.py --plan-dry-run --kv-page 64 --steps 2 --warmup 1 --requests 1024 > gpurun_out/c4_paged.json 2> gpurun_out/c4_paged.err; echo "c4 paged rc $?"
tail -2 gpurun_out/c4_paged.err
timeout 1500 python tools/config3.py > gpurun_out/r2_config3.json 2> gpurun_out/config3.err; echo "config3 rc $?"
tail -n 2 gpurun_out/config3.err

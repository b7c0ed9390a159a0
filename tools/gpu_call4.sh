# full GPU suite (paged RRA/WAA, early stream-K fixup), decode A/B, timelines, configs 3 and 4
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc $?"
tail -4 gpurun_out/pytest_gpu_full.log
timeout 600 python tools/ab_decode.py 0 128 0 128 > gpurun_out/ab_early_fixup.log 2>&1; echo "ab rc $?"
timeout 300 python tools/probe_timeline.py 64 20480 5120 > gpurun_out/tl_ffn1.log 2>&1
EXG_EXTRA_FLAGS=128 timeout 300 python tools/probe_timeline.py 64 20480 5120 > gpurun_out/tl_ffn1_noearly.log 2>&1; echo "tl rc $?"
timeout 1500 python bench.py --plan-dry-run --steps 3 --warmup 3 --requests 1024 > gpurun_out/c4_slots.json 2> gpurun_out/c4_slots.err; echo "c4 slots rc $?"
timeout 1500 python bench.py --plan-dry-run --kv-page 64 --steps 3 --warmup 3 --requests 1024 > gpurun_out/c4_paged.json 2> gpurun_out/c4_paged.err; echo "c4 paged rc $?"
timeout 1800 python tools/config3.py 1024 > gpurun_out/r2_config3_1024.json 2> gpurun_out/config3.err; echo "config3 rc $?"

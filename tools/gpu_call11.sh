# scheduler margin A/B on one box: the bench at --margin 0.03 (default) and 0.0
mkdir -p gpurun_out
timeout 1500 python bench.py --bounds headline --baseline-requests 0 --no-cpu-baseline --dyn 0 --margin 0.03 > gpurun_out/bench_m3.json 2> gpurun_out/bench_m3.err; echo "m3 rc $?"
timeout 1500 python bench.py --bounds headline --baseline-requests 0 --no-cpu-baseline --dyn 0 --margin 0.0 > gpurun_out/bench_m0.json 2> gpurun_out/bench_m0.err; echo "m0 rc $?"
timeout 1500 python bench.py --bounds headline --baseline-requests 0 --no-cpu-baseline --dyn 0 --margin 0.03 > gpurun_out/bench_m3b.json 2> gpurun_out/bench_m3b.err; echo "m3b rc $?"

# simulator fidelity with the in-situ decode attention table (diag) vs the default
mkdir -p gpurun_out
EXG_PROFILE_INSITU=1 timeout 1200 python tools/config3.py 1024 > gpurun_out/c3_insitu.json 2> gpurun_out/c3_insitu.err; echo "c3 insitu rc $?"
EXG_PROFILE_INSITU=1 timeout 1500 python bench.py --bounds headline --baseline-requests 0 --no-cpu-baseline --dyn 0 > gpurun_out/bench_insitu.json 2> gpurun_out/bench_insitu.err; echo "bench insitu rc $?"
timeout 1500 python bench.py --bounds headline --baseline-requests 0 --no-cpu-baseline --dyn 0 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc $?"

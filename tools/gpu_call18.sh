mkdir -p gpurun_out
timeout 1800 python tools/config3.py 1024 > gpurun_out/r2_config3_final.json 2> gpurun_out/config3.err; echo "config3 rc $?"
tail -2 gpurun_out/config3.err

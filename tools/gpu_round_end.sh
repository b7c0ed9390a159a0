# round-end evidence on one B200: bench line, ncu launch list of the timed
# step, ncu --set full per kernel class -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --bounds headline --baseline-requests 0 \
  --no-cpu-baseline --dyn 0 > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc $?"
timeout 900 bash tools/ncu_traffic.sh > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc $?"
ls gpurun_out

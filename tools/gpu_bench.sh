# one bench run (default flags) -> gpurun_out/bench_<tag>.json
mkdir -p gpurun_out
tag=${1:-run}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi_$tag.txt
timeout 1500 python bench.py ${@:2} > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc $?"
tail -2 gpurun_out/bench_$tag.err

# refresh configs 3-5 evidence with the current kernels
mkdir -p gpurun_out
timeout 1500 python tools/config3.py > gpurun_out/r1_config3.json 2> gpurun_out/config3.err; echo "config3 rc $?"
timeout 1500 python tools/plan_configs.py > gpurun_out/r1_plans.json 2> gpurun_out/plans.err; echo "plans rc $?"
tail -n 2 gpurun_out/config3.err; tail -n 2 gpurun_out/plans.err

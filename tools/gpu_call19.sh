mkdir -p gpurun_out
timeout 600 python tools/probe_t5_attn.py > gpurun_out/t5_attn.log 2>&1; echo "rc $?"
cat gpurun_out/t5_attn.log

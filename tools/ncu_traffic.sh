#!/bin/bash
# One `ncu --set full` capture per kernel class at a workload shape whose
# algorithmic bytes / flops are known exactly (OPT-13B, task S), for the
# bench's roofline.traffic (tools/kernel_traffic.py turns them into
# profiles/kernel_traffic.json).  Runs on the GPU box; writes gpurun_out/.
set -u
N="ncu --set full --clock-control none --import-source on -s 1 -c 1"
$N -k regex:gemm_pair -o gpurun_out/tr_prefill_gemm python tools/probe_kernels.py gemm 8192 15360 5120 pre
$N -k regex:gemm_tc -o gpurun_out/tr_decode_gemm python tools/probe_kernels.py gemm 64 20480 5120 dec
$N -k regex:gemm_tc -o gpurun_out/tr_decode_gemm_resid python tools/probe_kernels.py gemm 64 5120 5120 dec 2
$N -k regex:decode_attn -o gpurun_out/tr_decode_attn python tools/probe_kernels.py dattn 64 384
$N -k regex:fmha -o gpurun_out/tr_prefill_attn python tools/probe_kernels.py pattn 32 256

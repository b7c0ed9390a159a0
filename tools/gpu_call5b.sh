# round-end evidence on the final code (bench line, ncu launch list, ncu --set full per class)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
bash tools/gpu_round_end.sh

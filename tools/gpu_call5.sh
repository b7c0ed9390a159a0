# LN preload A/B, then the round-end evidence (bench line, ncu launch list, ncu --set full per class)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q > gpurun_out/pytest_subset.log 2>&1; echo "pytest subset rc $?"
tail -2 gpurun_out/pytest_subset.log
EXG_LN_PRELOAD=0 timeout 600 python tools/ab_decode.py 0 0 > gpurun_out/ab_ln_off.log 2>&1; echo "ab ln off rc $?"
EXG_LN_PRELOAD=1 timeout 600 python tools/ab_decode.py 0 0 > gpurun_out/ab_ln_on.log 2>&1; echo "ab ln on rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
bash tools/gpu_round_end.sh

mkdir -p gpurun_out
: > gpurun_out/fixup_ab.txt
for v in base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/fixup_ab.txt
  for s in "48 15360 5120 0" "48 5120 5120 2" "48 20480 5120 0" "48 5120 20480 2"; do
    timeout 120 python tools/probe_timeline.py $s | grep -A8 "rep 2" >> gpurun_out/fixup_ab.txt 2>&1
  done
done
for v in base new base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/fixup_ab.txt
  timeout 300 python tools/ab_decode.py 0 >> gpurun_out/fixup_ab.txt 2>&1
done
unset EXG_PROBE_LIB
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_fixup.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_fixup.log
grep -E "==|last_commit|epi_done|exit|event|tok_s" gpurun_out/fixup_ab.txt

mkdir -p gpurun_out
: > gpurun_out/hybrid_ab.txt
for v in base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/hybrid_ab.txt
  for s in "48 20480 5120 0" "48 50272 5120 3" "160 20480 5120 0"; do
    timeout 120 python tools/probe_timeline.py $s | grep -A8 "rep 2" >> gpurun_out/hybrid_ab.txt 2>&1
  done
done
for v in base new base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/hybrid_ab.txt
  timeout 300 python tools/ab_decode.py 0 >> gpurun_out/hybrid_ab.txt 2>&1
done
unset EXG_PROBE_LIB
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_hybrid.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_hybrid.log
grep -E "==|T=|last_commit|epi_done|tok_s" gpurun_out/hybrid_ab.txt

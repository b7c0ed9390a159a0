mkdir -p gpurun_out
: > gpurun_out/kvfuse_ab.txt
for v in base new base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/kvfuse_ab.txt
  timeout 300 python tools/ab_decode.py 0 >> gpurun_out/kvfuse_ab.txt 2>&1
done
unset EXG_PROBE_LIB
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_kvfuse.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_kvfuse.log
cat gpurun_out/kvfuse_ab.txt

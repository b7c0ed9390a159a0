# fused KV append A/B (decode phase, OPT-13B RRA) + end-to-end parity tests
mkdir -p gpurun_out
: > gpurun_out/append_ab.txt
for i in 1 2; do
  echo "== base" >> gpurun_out/append_ab.txt
  EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so timeout 300 python tools/ab_decode.py 0 >> gpurun_out/append_ab.txt 2>&1
  echo "== new" >> gpurun_out/append_ab.txt
  timeout 300 python tools/ab_decode.py 0 >> gpurun_out/append_ab.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_append.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_append.log
cat gpurun_out/append_ab.txt

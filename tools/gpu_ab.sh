# A/B of this build against another one (tools/_base/libexegpt.so, built from
# another commit): decode / encode phase times (tools/ab_decode.py), per-CTA
# decode GEMM timelines, prefill attention and CTA-pair GEMM probes; then the
# GPU test suite on this build.  Results -> gpurun_out/ab.txt
#   git stash; python -c "import __graft_entry__ as g; g.build()"; mkdir -p tools/_base
#   cp paper_2404_07947_b200/libexegpt.so tools/_base/; git stash pop; (rebuild)
#   gpurun -- 'bash tools/gpu_ab.sh'
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for v in base new base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/ab.txt
  timeout 300 python tools/ab_decode.py 0 >> gpurun_out/ab.txt 2>&1
done
for v in base new; do
  if [ $v = base ]; then export EXG_PROBE_LIB=$PWD/tools/_base/libexegpt.so; else unset EXG_PROBE_LIB; fi
  echo "== $v" >> gpurun_out/ab.txt
  for s in "48 15360 5120 0" "48 5120 5120 2" "48 20480 5120 0" "48 5120 20480 2"; do
    timeout 120 python tools/probe_timeline.py $s | grep -A8 "rep 2" >> gpurun_out/ab.txt 2>&1
  done
  timeout 300 python tools/probe_kernels.py pmix >> gpurun_out/ab.txt 2>&1
done
unset EXG_PROBE_LIB
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_ab.log

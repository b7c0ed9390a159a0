mkdir -p gpurun_out
: > gpurun_out/split_ab.txt
for v in 0 256 128 0 256 128; do
  echo "== split $v" >> gpurun_out/split_ab.txt
  EXG_DECODE_SPLIT=$v timeout 300 python tools/ab_decode.py 0 >> gpurun_out/split_ab.txt 2>&1
done
cat gpurun_out/split_ab.txt

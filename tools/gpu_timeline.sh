mkdir -p gpurun_out
for s in "48 15360 5120 0" "48 5120 5120 2" "48 20480 5120 0" "48 5120 20480 2"; do
  timeout 120 python tools/probe_timeline.py $s
done > gpurun_out/timeline.txt 2>&1
cat gpurun_out/timeline.txt | grep -A8 "rep 2"

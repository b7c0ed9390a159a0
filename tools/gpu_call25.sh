# decode-attention variants (ring depth / CTAs per SM) on the OPT-13B RRA decode phase
mkdir -p gpurun_out
for v in 0 1 3 16 0; do EXG_DECODE_STAGES=$v timeout 400 python tools/ab_decode.py 0 > gpurun_out/ab_stages_$v.log 2>&1; echo "stages $v"; cat gpurun_out/ab_stages_$v.log; done

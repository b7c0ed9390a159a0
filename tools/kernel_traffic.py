"""profiles/kernel_traffic.json from the `ncu --set full` captures of
tools/ncu_traffic.sh: DRAM bytes (read + write) per unit of the bench's
algorithmic work for each kernel class -- bytes per algorithmic byte for the
HBM-bound classes, bytes per flop for the tensor-bound ones -- so bench.py
can report roofline.traffic per launch.

    python tools/kernel_traffic.py gpurun_out   (reads tr_<class>.ncu-rep)

The work formulas are the engine's (engine.cu kend() calls) at the probe
shapes below."""
import csv
import io
import json
import os
import subprocess
import sys

H, DH = 40, 128
CASES = {
    # class: (report, work per launch, description)
    "prefill_gemm": ("tr_prefill_gemm", 2.0 * 8192 * 15360 * 5120, "QKV GEMM T=8192 N=15360 K=5120, flops"),
    "decode_gemm": ("tr_decode_gemm", 2.0 * 20480 * 5120 + 2.0 * 64 * 5120 + 2.0 * 64 * 20480,
                    "FFN1-shaped decode GEMM T=64 N=20480 K=5120, algorithmic bytes"),
    "decode_gemm_resid": ("tr_decode_gemm_resid", 2.0 * 5120 * 5120 + 2.0 * 64 * 5120 + 8.0 * 64 * 5120,
                          "O-proj decode GEMM (fp32 residual epilogue) T=64 N=K=5120, algorithmic bytes"),
    "decode_attn": ("tr_decode_attn", 64 * 384 * 2.0 * H * DH * 2.0 + 64 * H * DH * 2.0 * 2.0,
                    "decode attention B=64 rows x 384 keys, 40 heads, algorithmic bytes"),
    "prefill_attn": ("tr_prefill_attn", 4.0 * H * DH * 32 * 256 * 257 / 2,
                     "causal prefill attention 32 requests x 256 tokens, flops"),
}


def dram_bytes(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[units[i]]
        tot += float(vals[i].replace(",", "")) * scale
    t = hdr.index("gpu__time_duration.sum")
    tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}[units[t]]
    return tot, float(vals[t].replace(",", "")) * tscale


def main(d):
    res = {}
    for cls, (rep, work, desc) in CASES.items():
        p = os.path.join(d, rep + ".ncu-rep")
        if not os.path.exists(p):
            continue
        b, t = dram_bytes(p)
        res[cls] = {"dram_bytes_per_work": b / work, "dram_bytes": b, "work": work, "ncu_time_s": t,
                    "probe": desc, "report": rep}
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")

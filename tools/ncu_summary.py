"""Compact summary of an ncu report (run here, on the CPU box):

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [...]

Prints per kernel launch: duration, DRAM bytes read/written, DRAM and
tensor-pipe utilisation, L2 throughput, SM clock, occupancy, registers and
the top warp-stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_rt%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__cycles_elapsed.avg.per_second", "clk"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(path, ": no data")
        return
    hdr, units = rows[0], rows[1]
    idx = {n: i for i, n in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx.get("Kernel Name", 0)][:60]
        parts = []
        for k, short in KEYS:
            if k in idx and r[idx[k]] != "":
                parts.append("%s=%s%s" % (short, r[idx[k]], units[idx[k]] if units[idx[k]] not in ("", "%") else ""))
        stalls = []
        for n, i in idx.items():
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("%s | %s" % (name, " ".join(parts)))
        if stalls:
            print("    stalls: " + ", ".join("%s %.2f" % (s, v) for v, s in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        summarize(p)

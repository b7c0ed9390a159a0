"""Aggregate an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
per kernel: launches, total / average duration and share of the summed time.

    python tools/launch_summary.py launches.csv [title] > summary.txt

The per-launch times are cold-cache and serialised (ncu), so the shares, not
the absolute durations, are what the bench's live CUDA-event shares should
agree with."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def main(path, title=""):
    hdr = None
    agg = collections.OrderedDict()
    n = 0
    with open(path, newline="") as f:
        for r in csv.reader(f):
            if hdr is None:
                if "Kernel Name" in r and "Metric Value" in r:
                    hdr = {k: i for i, k in enumerate(r)}
                continue
            if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
                continue
            v = float(r[hdr["Metric Value"]].replace(",", "")) * SCALE[r[hdr["Metric Unit"]]]
            name = r[hdr["Kernel Name"]].split("(")[0]
            a = agg.setdefault(name, [0, 0.0])
            a[0] += 1
            a[1] += v
            n += 1
    tot = sum(a[1] for a in agg.values()) or 1.0
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)%s" %
          (": " + title if title else ""))
    print("launches %d, summed kernel time %.1f ms" % (n, tot / 1e3))
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-58s n=%7d sum=%11.1fus avg=%9.2fus share=%.3f" % (k[:58], c, t, t / c, t / tot))


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))

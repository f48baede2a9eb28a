"""Summarise an ncu launch list (ncu --metrics gpu__time_duration.sum --csv): per-kernel
launch count, total time and share of the profiled run."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            k = r[hdr.index("Kernel Name")].split("(")[0]
            us = float(r[hdr.index("Metric Value")].replace(",", "")) * SCALE[r[hdr.index("Metric Unit")]]
            agg[k][0] += 1
            agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-60s launches %4d  total %10.1f us  mean %8.1f us  share %5.1f%%" % (k[:60], n, t, t / n, 100 * t / tot))


if __name__ == "__main__":
    main(sys.argv[1])

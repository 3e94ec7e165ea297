"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per launch and per kernel."""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    return [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")) * scale[r[ui]]) for r in rows]


if __name__ == "__main__":
    L = load(sys.argv[1])
    if len(sys.argv) > 2 and sys.argv[2] == "all":
        for k, v in L:
            print("%10.1f us  %s" % (v, k))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in L:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in L)
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%10.1f us %5.1f%% %5d  %s" % (v, 100 * v / tot, n, k))
    print("%10.1f us total, %d launches" % (tot, len(L)))

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.
Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki][:70]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:70s} n={len(v):5d} avg={sum(v) / len(v):9.1f} us  share={sum(v) / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])

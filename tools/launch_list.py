"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch log into the
per-kernel launch list committed under profiles/ (cold-cache, serialised
per-launch times: compare kernel SHARES with the bench, not absolute times).

    python tools/launch_list.py gpurun_out/launches_c2.csv > profiles/r02/launches_c2.txt
"""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    h = rows[hdr]
    ik, iu, iv = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        unit = r[iu]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        name = r[ik].replace("(anonymous namespace)::", "").replace("wipes::", "")[:60]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    n = sum(a[0] for a in agg.values())
    print(f"# kernel launch list: {n} launches, {tot:.1f} us total (cold-cache, serialised)")
    print(f"{'kernel':<60} {'launches':>9} {'us total':>10} {'us/launch':>10} {'share':>7}")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:<60} {c:>9} {us:>10.1f} {us / c:>10.2f} {100 * us / tot:>6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])

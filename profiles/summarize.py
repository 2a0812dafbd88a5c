#!/usr/bin/env python
"""Summarise ncu evidence into committed text files.

    python profiles/summarize.py launches <launches.csv> > profiles/rNN/launches_<cfg>.txt
    python profiles/summarize.py kernel <prof.ncu-rep> > profiles/rNN/<kernel>_<cfg>.txt

`launches`: per-kernel totals and shares of the cold-cache, serialised launch
list (`ncu --metrics gpu__time_duration.sum`). `kernel`: the key counters of one
`ncu --set full` capture — duration, issue utilisation, pipe utilisation, DRAM
bytes (the roofline `traffic`), occupancy and the SASS opcode mix with stall
shares from the source page.
"""
import collections
import csv
import io
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    # skip ncu preamble lines until the header
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    iu = hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
        name = re.sub(r"wipes::<unnamed>::", "", name)
        v = float(r[iv].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "nsecond": 1e-3}.get(r[iu], 1.0)
        tot[name] += v * scale
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# kernel launch list: {sum(cnt.values())} launches, {T:.1f} us total (cold-cache, serialised)")
    print(f"{'kernel':60s} {'launches':>8s} {'us total':>10s} {'us/launch':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:10.2f} {100 * v / T:6.1f}%")


def kernel(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
            "sm__cycles_elapsed.avg.per_second"]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print("# ncu --set full capture")
        for k in keys:
            if k in d:
                print(f"{k:70s} {d[k]:>20s} {u.get(k, '')}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    kernels = []
    for x in rows:
        if x and x[0] == "Kernel Name":
            kernels.append([x[1] if len(x) > 1 else "?", None, []])
        elif x and x[0] == "Address" and kernels:
            kernels[-1][1] = x
        elif kernels and kernels[-1][1] is not None:
            kernels[-1][2].append(x)
    for name, h, body in kernels:
        ia, ie, iss = h.index("Source"), h.index("Instructions Executed"), \
            h.index("Warp Stall Sampling (All Samples)")
        by, st = collections.Counter(), collections.Counter()
        for x in body:
            if len(x) <= max(ia, ie, iss) or not x[ia].strip():
                continue
            toks = x[ia].strip().split()
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            by[op] += int(x[ie] or 0)
            st[op] += int(x[iss] or 0)
        T, S = sum(by.values()) or 1, sum(st.values()) or 1
        print(f"\n# SASS opcode mix of {name[:80]}: {T} warp instructions executed")
        for op, n in by.most_common(25):
            print(f"{op:12s} {n:12d} {100 * n / T:6.1f}%   stall-samples {100 * st[op] / S:5.1f}%")
    for row in r[2:]:
        d = dict(zip(hdr, row))
        stalls = {k.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", ""):
                  d[k] for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled_")
                  and k.endswith(".ratio")}
        if stalls:
            top = sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:8]
            print(f"\n# top warp stall reasons (cycles per issued instruction) {d.get('Kernel Name', '')[:60]}")
            for k, v in top:
                print(f"  {k:40s} {v}")


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel}[sys.argv[1]](sys.argv[2])

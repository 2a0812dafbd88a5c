"""Host->device copy probe (C2 step upload, 7.8 MB): a torch pin_memory()
buffer vs a buffer first touched by a thread bound to the GPU's NUMA node and
then pinned in place with cudaHostRegister; per-buffer NUMA page placement from
/proc/self/numa_maps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

n = 7798592 // 4
bus, cpus = bench.gpu_local_cpus(0)
print("gpu", bus, "local cpus", cpus[:4], "...", len(cpus))
if cpus:
    os.sched_setaffinity(0, cpus)
d = torch.empty(n, dtype=torch.float32, device="cuda")


def numa_of(ptr):
    best = None
    for line in open("/proc/self/numa_maps"):
        a = int(line.split()[0], 16)
        if a <= ptr and (best is None or a > best[0]):
            best = (a, line.strip())
    return " ".join(f for f in best[1].split() if f.startswith("N") or f.startswith("huge")) if best else "?"


def rate(h, label):
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{label} rep {rep}: {n * 4 / ms / 1e6:.1f} GB/s")


h1 = torch.empty(n, dtype=torch.float32).pin_memory()
print("torch pin_memory: pinned", h1.is_pinned(), "pages", numa_of(h1.data_ptr()))
rate(h1, "torch pin_memory")
a = np.empty(n, np.float32)
a.fill(1.0)  # first touch on this (node-bound) thread
h2 = torch.from_numpy(a)
err = torch.cuda.cudart().cudaHostRegister(h2.data_ptr(), n * 4, 0)
print("numpy + cudaHostRegister:", err, "pinned", h2.is_pinned(), "pages", numa_of(h2.data_ptr()))
rate(h2, "local+register")

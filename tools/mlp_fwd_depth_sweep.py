"""Fused forward time vs depth (inference): separates the per-tile fixed cost
(encoding, head, apply) from the per-layer cost. Usage: python tools/mlp_fwd_depth_sweep.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_12615_b200 import gen  # noqa: E402
from paper_2508_12615_b200.deform import Deformation  # noqa: E402

N = 300000
p = gen.gen3d(N, seed=0)
canon = {k: torch.from_numpy(v).cuda() for k, v in p.items()}
res = {}
for depth, lx, lt in ((1, 10, 6), (2, 10, 6), (4, 10, 6), (8, 10, 6), (1, 0, 0), (8, 0, 0)):
    d = Deformation(N, width=256, depth=depth, skip=-1, Lx=lx, Lt=lt)
    th = d.init_theta(0, head_scale=0.1)
    fr = d.forward(th, canon, [0.5], train=False)
    for _ in range(3):
        d.forward(th, canon, [0.5], fr, train=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        d.forward(th, canon, [0.5], fr, train=False)
    b.record()
    b.synchronize()
    res[f"D{depth}_L{lx}/{lt}"] = round(a.elapsed_time(b) / 10, 4)
print(json.dumps(res))

"""Tile-list length distribution of a config's frame (load-balance diagnostics):
    python tools/tile_lists.py c2"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_12615_b200 import gen  # noqa: E402
from paper_2508_12615_b200.raster import Rasterizer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = gen.make_config(name, seed=0)
dev = torch.device("cuda")
p = {k: torch.as_tensor(v, device=dev) for k, v in c["params"].items()}
kind = c["kind"]
r = Rasterizer(c["W"], c["H"], prim="2d" if kind == "2d" else "3d",
               blend="sum" if kind == "2d" else "alpha", device=dev)
r.forward(p, c.get("cams"), view_stride=c.get("view_stride", 0))
_, _, toff = r.bin_sort_outputs()
toff = toff.cpu().numpy().astype(np.int64)
L = np.diff(toff)
q = np.percentile(L, [50, 90, 99, 99.9, 100])
print(name, "tiles", L.size, "dups", int(L.sum()), "mean %.1f" % L.mean(),
      "p50/p90/p99/p99.9/max", q.astype(int).tolist(),
      "top-1%% share of dups %.3f" % (np.sort(L)[-max(1, L.size // 100):].sum() / max(1, L.sum())))

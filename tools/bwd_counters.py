"""Diagnostic: per-record work counters of the render backward (build with
-DWIPES_BWD_COUNT --out=variants/bcount.so; run with WIPES_LIB pointing at it).
Usage: python tools/bwd_counters.py c2|c3|c5"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_12615_b200 import abi, gen  # noqa: E402
from paper_2508_12615_b200.raster import Rasterizer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = gen.make_config(name)
dev = torch.device("cuda")
r = Rasterizer(c["W"], c["H"], prim="2d" if c["kind"] == "2d" else "3d", blend=c["blend"], device=dev)
params = {k: torch.from_numpy(v).to(dev) for k, v in c["params"].items()}
dL = torch.from_numpy(gen.gen_dLdC(c["B"], c["H"], c["W"], seed=0)).to(dev)
r.forward(params, c["cams"], c["view_stride"])
lib = abi.lib()
f = lib.wipes_debug_bwd_counters
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
f(buf, 1)
r.backward(dL)
torch.cuda.synchronize()
f(buf, 1)
staged, anyh, slots, red, lanes, chunks = [buf[i] for i in (0, 1, 2, 3, 4, 5)]
print(f"{name}: chunks {chunks}  staged records {staged}  with a slot hit {anyh} ({anyh / max(staged, 1):.2f})"
      f"  reduced {red} ({red / max(anyh, 1):.2f} of hit)  slots/hit-record {slots / max(anyh, 1):.2f}"
      f"  lane efficiency {lanes / max(32 * slots, 1):.2f}")

"""Exercise every kernel path once on small inputs (for compute-sanitizer):
2D SUM/ALPHA x {Sigma, Cholesky, RS} x tile {8, 16, 32}, 3D and 6D mini
configs, forward + backward, stats and parity copies."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_12615_b200 import gen  # noqa: E402
from paper_2508_12615_b200.raster import Rasterizer  # noqa: E402


def dev(p):
    return {k: torch.from_numpy(v).cuda() for k, v in p.items()}


def run2d():
    H, W = 72, 56
    for cov in ("sigma", "cholesky", "rs"):
        for blend in ("sum", "alpha"):
            for tile in (8, 16, 32):
                p = dev(gen.gen2d(H, W, 300, seed=1, cov_mode=cov, phase=True, depth=True,
                                  alpha=(0.2, 1.0)))
                r = Rasterizer(W, H, prim="2d", blend=blend, cov2=cov, tile=tile)
                r.forward(p)
                r.backward(torch.rand(1, 3, H, W, device="cuda") - 0.5)
                r.render_stats()
                r.bin_sort_outputs()
                r.get_preprocess()
                r.get_grad_moments()


def run3d():
    for name in ("p3d", "p6d"):
        c = gen.make_config(name, seed=0, N=3000)
        r = Rasterizer(c["W"], c["H"], prim="3d", blend="alpha")
        r.forward(dev(c["params"]), c["cams"], c["view_stride"])
        r.backward(torch.rand(c["B"], 3, c["H"], c["W"], device="cuda") - 0.5)
        r.render_stats()
        r.bin_sort_outputs()


if __name__ == "__main__":
    run2d()
    run3d()
    torch.cuda.synchronize()
    print("sanitize_run: ok")

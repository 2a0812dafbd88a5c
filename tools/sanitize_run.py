"""Exercise every kernel path once on small inputs (for compute-sanitizer or
the WIPES_CHECKS device-assert build): 2D SUM/ALPHA x {Sigma, Cholesky, RS} x
tile {8, 16, 32} x {atomic, deterministic} backward, 3D and 6D mini configs
(paper / exact projection, RGB / SH colour), the fitting step, the tcgen05
GEMM and the deformation MLP; forward + backward, stats and parity copies."""
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
        for proj, sh, det in (("paper", None, 0), ("exact", None, 1), ("paper", 3, 0),
                              ("exact", 2, 1)):
            c = gen.make_config(name, seed=0, N=3000, sh_degree=sh)
            r = Rasterizer(c["W"], c["H"], prim="3d", blend="alpha", proj=proj, sh_degree=sh,
                           deterministic=det)
            r.forward(dev(c["params"]), c["cams"], c["view_stride"])
            r.backward(torch.rand(c["B"], 3, c["H"], c["W"], device="cuda") - 0.5)
            r.render_stats()
            r.bin_sort_outputs()


def run_next():
    from paper_2508_12615_b200 import abi
    from paper_2508_12615_b200.deform import Deformation
    from paper_2508_12615_b200.train import Fitter2D
    tgt = gen.smooth_target(48, 40, seed=0)
    p = gen.init2d_from_target(tgt, 200, seed=0)
    for det in (0, 1):
        f = Fitter2D(torch.from_numpy(tgt).cuda(), dev(p), deterministic=det)
        f.fit(5, check_every=5)
    d = Deformation(1000)
    th = d.init_theta(0)
    q = gen.gen3d(1000, seed=0)
    canon = dev(q)
    fr = d.forward(th, canon, [0.0, 0.5])
    d.backward(th, canon, {k: torch.randn_like(fr[k]) for k in ("mean", "quat", "scale", "freq")})
    d.forward(th, canon, [0.0, 0.5], train=False)  # the fused on-chip forward
    # 20,000 rows (157 tiles, ragged): multi-tile rings of the fused layer backward
    d2 = Deformation(10000)
    th2 = d2.init_theta(1)
    c2 = dev(gen.gen3d(10000, seed=2))
    fr2 = d2.forward(th2, c2, [0.25, 0.75])
    d2.backward(th2, c2, {k: torch.randn_like(fr2[k]) for k in ("mean", "quat", "scale", "freq")})
    d2.forward(th2, c2, [0.25, 0.75], train=False)
    for amn in (False, True):
        for bmn in (False, True):
            A = torch.randn(304, 136, device="cuda").to(torch.bfloat16)
            B = torch.randn(72, 136, device="cuda").to(torch.bfloat16)
            A2 = A.t().contiguous() if amn else A
            B2 = B.t().contiguous() if bmn else B
            C = torch.zeros(304, 72, device="cuda")
            abi.gemm(A2, B2, C, 304, 72, 136, 304 if amn else 136, 72 if bmn else 136, 72,
                     epilogue="atomic_f32", a_mn=amn, b_mn=bmn, split_k=3)


if __name__ == "__main__":
    # argv: any of 2d 3d next (default all) — racecheck is run on the
    # rasterizer parts only (its shared-memory hazard tracking is slow)
    parts = sys.argv[1:] or ["2d", "3d", "next"]
    if "2d" in parts:
        run2d()
    if "3d" in parts:
        run3d()
    if "next" in parts:
        run_next()
    torch.cuda.synchronize()
    print("sanitize_run: ok")

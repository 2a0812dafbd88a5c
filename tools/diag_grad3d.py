"""Diagnostic: strict (exclude-and-count) gradient parity of the 3D/6D paths
against the oracle, printing every violation with its context (GPU needed).
Usage: python tools/diag_grad3d.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as ora  # noqa: E402
from paper_2508_12615_b200 import gen  # noqa: E402
from parity_util import (oracle_cfg, gpu_rasterizer, to_dev, pixel_violations,  # noqa: E402
                         ambiguous_rows, GRAD_ATOL, GRAD_RTOL, KAPPA, oracle_grads)


def px(a):
    return np.asarray(a).transpose(0, 2, 3, 1).reshape(-1, 3)


def run(name, blend="alpha", seed=0, dseed=1, **kw):
    extra = {}
    ok = {}
    if kw.get("proj") == "exact":
        extra["proj"] = "exact"
        ok["exact_proj"] = True
    if kw.get("sh") is not None:
        extra["sh_degree"] = kw["sh"]
        ok["sh_degree"] = kw["sh"]
    if kw.get("det"):
        extra["deterministic"] = 1
    c = gen.make_config(name, seed=seed, **({"sh_degree": kw["sh"]} if kw.get("sh") is not None else {}))
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True, **ok)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    r = gpu_rasterizer("3d", H, W, blend, **extra)
    out = r.forward(to_dev(p), cams, vs)
    dL = gen.gen_dLdC(B, H, W, seed=dseed)
    g = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    ro = ora.render(cfg_o, pr, dLdC=px(dL))
    nbp, namb = pixel_violations(px(out["image"].cpu().numpy()), ro["color"], ro["margin"])
    ro = ora.render(cfg_o, pr, dLdC=px(dL), abs_terms=True)
    og, og_abs = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    print(f"== {name} {blend} {kw} : pixel viol {nbp}, ambiguous px {namb}, excluded rows {exc.sum()}")
    for k, ref in og.items():
        if k not in g:
            continue
        got = g[k].cpu().numpy().astype(np.float64)
        ref = np.asarray(ref)
        keep = ~exc
        err = np.abs(got - ref)
        tol = np.maximum(GRAD_ATOL, GRAD_RTOL * np.abs(ref))
        bad_plain = (err > tol).reshape(err.shape[0], -1).any(1) & keep
        tol = np.maximum(tol, KAPPA * np.asarray(og_abs[k]))
        bad = (err > tol)
        print(f"  {k:8s} plain-tolerance rows viol kept {int(bad_plain.sum())}; "
              f"max err/S {np.max(err[keep] / np.maximum(np.asarray(og_abs[k])[keep], 1e-300)):.2e}")
        rows_bad = bad.reshape(bad.shape[0], -1).any(1)
        nb_keep = int((rows_bad & keep).sum())
        nb_exc = int((rows_bad & ~keep).sum())
        print(f"  {k:8s} rows viol kept {nb_keep:4d}  excluded {nb_exc:4d}  "
              f"max |ref| {np.abs(ref).max():.3e}")
        idx = np.nonzero((bad.reshape(bad.shape[0], -1)) & keep[:, None])
        ga = got.reshape(got.shape[0], -1)
        ra = ref.reshape(ref.shape[0], -1)
        aa = np.asarray(og_abs[k]).reshape(ref.shape[0], -1) if k in og_abs else ra
        for (i, j) in list(zip(*idx))[:12]:
            print(f"    row {i} comp {j}: got {ga[i, j]: .6e} ref {ra[i, j]: .6e} "
                  f"rel {abs(ga[i, j] - ra[i, j]) / max(abs(ra[i, j]), 1e-30):.2e} "
                  f"S {abs(aa[i, j]):.3e}")
    sys.stdout.flush()


if __name__ == "__main__":
    torch.cuda.init()
    from paper_2508_12615_b200 import build
    if not os.environ.get("WIPES_LIB"):
        build.build()
    ora.build()
    print("library:", os.environ.get("WIPES_LIB", "in-tree"))
    run("p3d", "alpha")
    run("p3d", "sum")
    run("p6d", "alpha")
    if "quick" in sys.argv:
        sys.exit(0)
    if "seeds" in sys.argv:
        for ds in (11, 12, 13):
            run("p3d", "alpha", dseed=ds)
            run("p3d", "sum", dseed=ds)
            run("p6d", "alpha", seed=1, dseed=ds)
        sys.exit(0)
    run("p3d", "alpha", proj="exact", dseed=2)
    run("p3d", "sum", proj="exact", dseed=2)
    run("p6d", "alpha", proj="exact", dseed=2)
    run("p3d", "alpha", sh=3, dseed=4)
    run("p3d", "sum", sh=2, dseed=4)
    run("p6d", "alpha", sh=3, dseed=4)
    run("p3d", "alpha", seed=1, dseed=7, det=True)

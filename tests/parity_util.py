"""Helpers shared by the parity tests: run the CUDA path (through the C ABI via
paper_2508_12615_b200.raster) and the oracle on the same seeded float32 inputs.
The oracle never sees any CUDA output; tolerances follow DESIGN.md R23."""
from __future__ import annotations

import numpy as np

PIX_ATOL, PIX_RTOL = 1e-5, 1e-4      # north_star: pixels 1e-5 abs / 1e-4 rel
GRAD_ATOL, GRAD_RTOL = 1e-5, 1e-3    # north_star: gradients 1e-3 rel, 1e-5 abs floor
AMBIG = 1e-5                          # decision margin below which a pixel is masked

F32 = np.float32


def f32(x):
    return float(np.float32(x))


def oracle_cfg(ora, kind, H, W, blend, tile=16, cov2="sigma", use_rect=False, **kw):
    prim3d = kind != "2d"
    return ora.Cfg(width=W, height=H, tile=tile, prim3d=prim3d, alpha_blend=(blend == "alpha"),
                   cov2=cov2, use_rect=use_rect,
                   dilation=f32(0.3) if prim3d else 0.0, **kw)


def gpu_rasterizer(kind, H, W, blend, tile=16, cov2="sigma", **kw):
    from paper_2508_12615_b200.raster import Rasterizer
    return Rasterizer(W, H, prim="2d" if kind == "2d" else "3d", blend=blend, cov2=cov2,
                      tile=tile, **kw)


def to_dev(params, device="cuda"):
    import torch
    return {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(device)
            for k, v in params.items()}


def pixel_violations(got, ref, margin=None):
    """Element-wise |g - o| <= max(atol, rtol |o|); pixels with decision margin
    < AMBIG are masked (either outcome is correct, R24)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = np.maximum(PIX_ATOL, PIX_RTOL * np.abs(ref))
    bad = np.abs(got - ref) > tol
    if margin is not None:
        amb = margin < AMBIG
        if bad.ndim > amb.ndim:
            amb = amb.reshape(amb.shape + (1,) * (bad.ndim - amb.ndim))
        bad = bad & ~amb
        return int(bad.sum()), int((margin < AMBIG).sum())
    return int(bad.sum()), 0


def grad_violations(got, ref, atol=GRAD_ATOL, rtol=GRAD_RTOL):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = np.maximum(atol, rtol * np.abs(ref))
    bad = np.abs(got - ref) > tol
    return int(bad.sum()), float(np.max(np.abs(got - ref) - tol, initial=-1.0))

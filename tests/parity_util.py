"""Helpers shared by the parity tests: run the CUDA path (through the C ABI via
paper_2508_12615_b200.raster) and the oracle on the same seeded float32 inputs.
The oracle never sees any CUDA output; tolerances follow DESIGN.md R23."""
from __future__ import annotations

import numpy as np

PIX_ATOL, PIX_RTOL = 1e-5, 1e-4      # north_star: pixels 1e-5 abs / 1e-4 rel
GRAD_ATOL, GRAD_RTOL = 1e-5, 1e-3    # north_star: gradients 1e-3 rel, 1e-5 abs floor
AMBIG = 1e-5                          # decision margin below which a pixel is masked
# DESIGN.md R23b: the per-pair evaluation on the FP32/SFU pipes the north star
# prescribes carries an error of at most KAPPA of each term's magnitude (MUFU
# sin/cos absolute error 2^-20.5 plus the FP32 rounding of theta and of its
# RZ scaling to revolutions for |theta| <= 60 rad, ex2 relative 2^-22, FP32
# products and sums), so an element whose terms cancel to below ~KAPPA/1e-3 of
# their magnitude S cannot meet 1e-3 relative: its tolerance is KAPPA * S.
KAPPA = 2.0 ** -17

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


def ambiguous_rows(pr, margin, B, N, H, W, view_stride=0, pix=None, alpha_min=1.0 / 255.0):
    """SURVEY §8(c) parity protocol: the gradient rows that have a pair at a
    masked (decision margin < AMBIG) pixel — those may legitimately differ
    (R24) and are excluded and counted; every other row must meet
    the tolerance with zero violations. A pair can influence a pixel only if
    alpha*W >= alpha_min there (R8); since W <= G, the rows excluded are those
    whose oracle record has alpha*G >= alpha_min*(1 - 1e-3) at a masked pixel of
    their view (a superset of the pairs evaluated at that pixel, in front of or
    behind an ambiguous termination alike). Rows are primitives for a shared
    scene (view_stride = 0) and (view, primitive) for per-frame sets. `pix`
    gives the flat pixel ids of `margin` when only a sample was rendered.
    Returns a bool mask [rows] of excluded rows."""
    margin = np.asarray(margin)
    ids = np.nonzero(margin < AMBIG)[0]
    if pix is not None:
        ids = np.asarray(pix)[ids]
    mux, muy = pr.field("mux").reshape(B, N), pr.field("muy").reshape(B, N)
    a, b, c = (pr.field(k).reshape(B, N) for k in ("a", "b", "c"))
    al = pr.field("alpha").reshape(B, N)
    live = np.asarray(pr.flag).reshape(B, N) == 0
    touch = np.zeros((B, N), bool)
    thr = alpha_min * (1.0 - 1e-3)
    with np.errstate(over="ignore", invalid="ignore"):
        for pid in ids:
            v, rem = int(pid // (H * W)), int(pid % (H * W))
            dx = (rem % W) + 0.5 - mux[v]
            dy = (rem // W) + 0.5 - muy[v]
            q = a[v] * dx * dx + 2.0 * b[v] * dx * dy + c[v] * dy * dy
            touch[v] |= live[v] & (al[v] * np.exp(-0.5 * q) >= thr)
    return touch.any(0) if view_stride == 0 else touch.reshape(-1)


def oracle_grads(ora, cfg, p, pr, ro, cams=None, view_stride=0):
    """Oracle parameter gradients and their running-error-bound scales S
    (oracle.grad_bound on render(..., abs_terms=True) output)."""
    if cfg.prim3d:
        og = ora.chain3d(cfg, p, cams, pr, ro["rgrad"], view_stride=view_stride)
    else:
        og = ora.chain2d(cfg, p, pr, ro["rgrad"])
    bound = ora.grad_bound(cfg, p, pr, ro["rgrad_abs"], cams, view_stride)
    return og, bound


def check_grads_strict(got: dict, ref: dict, excluded, label="", keys=None, bound=None):
    """Apply the SURVEY §8(c) protocol to every gradient group: zero
    violations on the rows not excluded of |g - o| <= max(1e-5, 1e-3 |o|,
    KAPPA * S) — the north-star tolerance, widened only for elements whose
    terms cancel below FP32/SFU evaluation accuracy (S = `bound`, DESIGN.md
    R23b). Prints, per group, the violations of the plain north-star form and
    of the full form (must be 0) and the excluded rows; returns them."""
    out = {}
    keep = ~np.asarray(excluded, bool)
    for k in (keys or ref.keys()):
        if k not in got or k not in ref:
            continue
        g = got[k]
        g = g.detach().cpu().numpy() if hasattr(g, "detach") else np.asarray(g)
        g = np.asarray(g, np.float64)[keep]
        o = np.asarray(ref[k], np.float64)[keep]
        err = np.abs(g - o)
        tol = np.maximum(GRAD_ATOL, GRAD_RTOL * np.abs(o))
        plain = int((err > tol).sum())
        if bound is not None:
            tol = np.maximum(tol, KAPPA * np.asarray(bound[k], np.float64)[keep])
        full = int((err > tol).sum())
        out[k] = (full, plain, float(np.max(err - tol, initial=-1.0)))
    rows = len(np.asarray(excluded))
    print(f"[parity] {label}: rows {rows}, excluded {int(np.sum(excluded))}; "
          + ", ".join(f"{k} {v[0]} viol ({v[1]} beyond 1e-3 rel / 1e-5 abs)"
                      for k, v in out.items()))
    bad = {k: v for k, v in out.items() if v[0]}
    assert not bad, f"{label}: gradient violations on non-excluded rows: {bad}"
    return out

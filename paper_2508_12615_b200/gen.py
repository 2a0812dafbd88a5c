"""Seeded synthetic input generators for the WIPES rasterizer.

This module serves BOTH the CUDA path (bench.py, GPU tests) and the oracle
(tests, cpu_baseline). It holds none of the method's arithmetic: it only draws
random parameters (numpy PCG64, float64 draws cast once to float32) and builds
pinhole cameras. The recipes follow SURVEY.md §8(d):
shapes and distributions shaped like the paper's workloads — Kodak-sized 2D
fitting (Sec. 5.1), Mip-NeRF360-like static scenes (Table 3 point
counts) and dynamic per-frame scenes (Eq. 8).
The only distribution the paper fixes is "frequency coefficients ... randomly
initialized with a normal distribution"; all else is a proposal.
"""
from __future__ import annotations

import math

import numpy as np

F32 = np.float32


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# --------------------------------------------------------------------------
# 2D image-fitting primitives (Eq. 4 weighted sum; Cholesky / RS)
# --------------------------------------------------------------------------
def gen2d(H: int, W: int, N: int, seed: int = 0, cov_mode: str = "sigma",
          freq_std: float = 0.5, phase: bool = False, color_max: float = 0.1,
          alpha=1.0, s0: float | None = None, depth: bool = False) -> dict:
    """N 2D wavelet primitives on an H x W image.

    mean ~ U[0,W) x U[0,H); per-axis envelope std s0*exp(N(0, 0.5^2)) with
    s0 = sqrt(H W / N) (area equipartition); orientation
    theta ~ U[0, pi). The covariance is drawn directly in the requested
    parameterisation (no covariance arithmetic here):
      sigma    : (sxx, sxy, syy) = (sx^2, rho sx sy, sy^2), rho ~ U(-0.8, 0.8)
      cholesky : (l1, l2, l3) = (sx, rho sy, sqrt(1-rho^2) sy)
      rs       : (theta, sx, sy)
    freq ~ N(0, freq_std^2) rad/px per axis; phase ~ U[-pi, pi) if requested;
    colour ~ U[0, color_max)^3; alpha = constant or U[lo, hi).
    """
    g = _rng(seed)
    if s0 is None:
        s0 = math.sqrt(H * W / N)
    mean = np.stack([g.uniform(0, W, N), g.uniform(0, H, N)], 1)
    sx = s0 * np.exp(g.normal(0, 0.5, N))
    sy = s0 * np.exp(g.normal(0, 0.5, N))
    th = g.uniform(0, math.pi, N)
    rho = g.uniform(-0.8, 0.8, N)
    if cov_mode == "sigma":
        cov = np.stack([sx * sx, rho * sx * sy, sy * sy], 1)
    elif cov_mode == "cholesky":
        cov = np.stack([sx, rho * sy, np.sqrt(1 - rho * rho) * sy], 1)
    elif cov_mode == "rs":
        cov = np.stack([th, sx, sy], 1)
    else:
        raise ValueError(cov_mode)
    freq = g.normal(0, freq_std, (N, 2))
    ph = g.uniform(-math.pi, math.pi, N) if phase else None
    color = g.uniform(0, color_max, (N, 3))
    if isinstance(alpha, tuple):
        op = g.uniform(alpha[0], alpha[1], N)
    else:
        op = np.full(N, float(alpha))
    out = dict(mean=mean, cov=cov, freq=freq, color=color, opacity=op)
    if ph is not None:
        out["phase"] = ph
    if depth:
        out["depth"] = g.uniform(1.0, 10.0, N)
    return {k: np.ascontiguousarray(v.astype(F32)) for k, v in out.items()}


# --------------------------------------------------------------------------
# 3D scenes and cameras (Eq. 3 alpha blending)
# --------------------------------------------------------------------------
def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0)):
    """World->camera (R, t) for a camera at `eye` looking at `target`;
    camera axes x right, y down, z forward (OpenCV convention)."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd], 0)
    t = -R @ eye
    return R, t


def camera(eye, W, H, focal_frac=0.9, target=(0, 0, 0), near=0.01, far=100.0):
    R, t = look_at(eye, target)
    f = focal_frac * W
    return dict(R=R.astype(F32), t=t.astype(F32), fx=float(F32(f)), fy=float(F32(f)),
                cx=float(F32(W / 2)), cy=float(F32(H / 2)), near=float(F32(near)),
                far=float(F32(far)), width=W, height=H)


def ring_cameras(B, W, H, radius=3.0, height=0.5, focal_frac=0.9, phase0=0.0):
    cams = []
    for v in range(B):
        a = phase0 + 2 * math.pi * v / B
        eye = (radius * math.cos(a), -height, radius * math.sin(a))
        cams.append(camera(eye, W, H, focal_frac))
    return cams


def gen3d(N: int, seed: int = 0, scale_med: float = 0.004, scale_mult: float = 1.0,
          inner_frac: float = 0.7, phase: bool = False, sh_degree=None) -> dict:
    """Mip-NeRF360-like synthetic scene: 70% of centres
    volume-uniform in a ball r in [0.2, 1], 30% on a shell r in [8, 20];
    per-axis scale scale_med*exp(N(0, 0.7^2)) (shell scaled by r/3);
    q ~ N(0, I4); opacity bimodal (40% U[0,0.2), 60% U[0.6,1.0));
    colour U[0,1)^3; frequency n / mean-scale, n ~ N(0, I3) (about 1 rad per sigma)."""
    g = _rng(seed)
    n_in = int(round(inner_frac * N))
    d = g.normal(size=(N, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = np.empty(N)
    u = g.uniform(0, 1, N)
    r[:n_in] = (0.2 ** 3 + u[:n_in] * (1.0 - 0.2 ** 3)) ** (1 / 3)
    r[n_in:] = g.uniform(8.0, 20.0, N - n_in)
    mean = d * r[:, None]
    scale = scale_med * scale_mult * np.exp(g.normal(0, 0.7, (N, 3)))
    scale[n_in:] *= (r[n_in:] / 3.0)[:, None]
    quat = g.normal(size=(N, 4))
    pick = g.uniform(0, 1, N) < 0.4
    op = np.where(pick, g.uniform(0, 0.2, N), g.uniform(0.6, 1.0, N))
    color = g.uniform(0, 1, (N, 3))
    freq = g.normal(size=(N, 3)) / scale.mean(axis=1, keepdims=True)
    out = dict(mean=mean, scale=scale, quat=quat, freq=freq, color=color, opacity=op)
    if phase:
        out["phase"] = g.uniform(-math.pi, math.pi, N)
    if sh_degree is not None:
        # NEXT-3 colour coefficients [N, (deg+1)^2, 3]: DC term U(-1.5, 1.5),
        # band l >= 1 ~ N(0, (0.25 / l)^2) (a 3DGS-like spectrum; no SH arithmetic here)
        K = (sh_degree + 1) ** 2
        sh = np.empty((N, K, 3))
        sh[:, 0, :] = g.uniform(-1.5, 1.5, (N, 3))
        for l in range(1, sh_degree + 1):
            sh[:, l * l:(l + 1) * (l + 1), :] = g.normal(0, 0.25 / l, (N, 2 * l + 1, 3))
        out["sh"] = sh
        del out["color"]
    return {k: np.ascontiguousarray(v.astype(F32)) for k, v in out.items()}


def gen6d(N: int, frames: int, seed: int = 0, scale_med: float = 0.006,
          scale_mult: float = 1.0, sh_degree=None) -> dict:
    """Per-frame ('time-conditioned') parameters: a stand-in for the deformation
    field F_theta of Eq. 8 — the MLP itself is out of scope:
    mu_t = mu + 0.02 sin(2 pi t/T + psi) v, f_t = f (1 + 0.1 sin(.)),
    s_t = s exp(0.05 sin(.)). Returned arrays are [frames*N, k] (view_stride = N)."""
    base = gen3d(N, seed, scale_med=scale_med, scale_mult=scale_mult, sh_degree=sh_degree)
    g = _rng(seed + 7919)
    psi = g.uniform(0, 2 * math.pi, N)
    vdir = g.normal(size=(N, 3))
    out = {k: [] for k in base}
    for t in range(frames):
        s = np.sin(2 * math.pi * t / max(frames, 1) + psi)
        out["mean"].append(base["mean"].astype(np.float64) + 0.02 * s[:, None] * vdir)
        out["freq"].append(base["freq"].astype(np.float64) * (1 + 0.1 * s)[:, None])
        out["scale"].append(base["scale"].astype(np.float64) * np.exp(0.05 * s)[:, None])
        for k in ("quat", "color", "opacity", "sh"):
            if k in base:
                out[k].append(base[k])
    return {k: np.ascontiguousarray(np.concatenate(v, 0).astype(F32)) for k, v in out.items()}


def arc_cameras(B, W, H, radius=2.5, focal_frac=0.9):
    """One monocular camera per frame on a 90-degree arc (D-NeRF style)."""
    cams = []
    for v in range(B):
        a = -math.pi / 4 + (math.pi / 2) * v / max(B - 1, 1)
        eye = (radius * math.sin(a), -0.3, -radius * math.cos(a))
        cams.append(camera(eye, W, H, focal_frac))
    return cams


def gen_dLdC(B: int, H: int, W: int, seed: int = 0) -> np.ndarray:
    """Upstream gradient dL/dC ~ U(-1, 1), planar [B, 3, H, W] float32."""
    return _rng(seed + 104729).uniform(-1, 1, (B, 3, H, W)).astype(F32)


# --------------------------------------------------------------------------
# NEXT-2 fitting inputs: a synthetic target and the SPEC's initialisation
# --------------------------------------------------------------------------
def zone_plate(H: int, W: int, k: float = 60.0) -> np.ndarray:
    """SPEC S:422-427 gen_zone_plate: I = 1/2 + 1/2 sin(k (u^2 + v^2)) with
    u, v in [-1, 1] at pixel centres, replicated to 3 channels -> [3, H, W]."""
    u = (np.arange(W) + 0.5) / W * 2.0 - 1.0
    v = (np.arange(H) + 0.5) / H * 2.0 - 1.0
    img = 0.5 + 0.5 * np.sin(k * (u[None, :] ** 2 + v[:, None] ** 2))
    return np.ascontiguousarray(np.broadcast_to(img, (3, H, W)).astype(F32))


def smooth_target(H: int, W: int, seed: int = 0, octaves: int = 5) -> np.ndarray:
    """A natural-image-like [3, H, W] target in [0, 1]: a sum of random
    sinusoidal gratings with 1/f amplitudes (no dataset is available)."""
    g = _rng(seed)
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    img = np.zeros((3, H, W))
    for o in range(octaves):
        for _ in range(4):
            f = (2.0 ** o) * 2 * math.pi / max(H, W) * g.uniform(0.5, 1.5)
            th = g.uniform(0, math.pi)
            ph = g.uniform(0, 2 * math.pi)
            wave = np.sin(f * (x * math.cos(th) + y * math.sin(th)) + ph)
            img += (0.5 ** o) * g.uniform(0.2, 1.0, 3)[:, None, None] * wave
    img -= img.min()
    img /= max(img.max(), 1e-12)
    return np.ascontiguousarray(img.astype(F32))


def init2d_from_target(target: np.ndarray, N: int, seed: int = 0, cov_mode: str = "cholesky",
                       freq_std: float = 0.05, phase: bool = False) -> dict:
    """SPEC S:328-331 init_primitives: positions uniform over the image; colours
    bilinearly sampled from the target at each position; opacity_raw = 0;
    covariance parameters giving Sigma = diag(s^2, s^2), s = sqrt(W H / N);
    freq ~ N(0, freq_std^2) per axis (rad/px). Returns raw float32 params."""
    C_, H, W = target.shape
    if N > H * W:
        raise ValueError("ImageTooSmall: N exceeds the pixel count")
    g = _rng(seed)
    mean = np.stack([g.uniform(0, W, N), g.uniform(0, H, N)], 1)
    # bilinear sample at the position (pixel centres at integer + 0.5)
    xs = np.clip(mean[:, 0] - 0.5, 0, W - 1)
    ys = np.clip(mean[:, 1] - 0.5, 0, H - 1)
    x0 = np.floor(xs).astype(np.int64)
    y0 = np.floor(ys).astype(np.int64)
    x1 = np.minimum(x0 + 1, W - 1)
    y1 = np.minimum(y0 + 1, H - 1)
    fx, fy = xs - x0, ys - y0
    t = target.astype(np.float64)
    color = ((1 - fx) * (1 - fy) * t[:, y0, x0] + fx * (1 - fy) * t[:, y0, x1]
             + (1 - fx) * fy * t[:, y1, x0] + fx * fy * t[:, y1, x1]).T
    s = math.sqrt(W * H / N)
    if cov_mode == "sigma":
        cov = np.tile([s * s, 0.0, s * s], (N, 1))
    elif cov_mode == "cholesky":
        cov = np.tile([s, 0.0, s], (N, 1))
    elif cov_mode == "rs":
        cov = np.tile([0.0, s, s], (N, 1))
    else:
        raise ValueError(cov_mode)
    out = dict(mean=mean, cov=cov, freq=g.normal(0, freq_std, (N, 2)), color=color,
               opacity=np.zeros(N))
    if phase:
        out["phase"] = np.zeros(N)
    return {k: np.ascontiguousarray(v.astype(F32)) for k, v in out.items()}


# --------------------------------------------------------------------------
# Named configurations (BASELINE.json configs)
# --------------------------------------------------------------------------
CONFIGS = {
    "c1": dict(kind="2d", H=64, W=64, N=256, blend="sum",
               desc="2D image fit: synthetic 64x64 RGB, 256 2D wavelet primitives"),
    "c2": dict(kind="2d", H=512, W=768, N=70000, blend="sum",
               desc="2D image fit: Kodak-shaped 768x512 RGB, 70k primitives, weighted sum"),
    "c3": dict(kind="3d", H=1080, W=1920, N=1000000, B=8, blend="alpha",
               desc="3D static NVS: 1M 3D wavelet primitives, 8 x 1080p views, alpha blending"),
    "c4": dict(kind="6d", H=1014, W=1352, N=300000, B=100, blend="alpha",
               desc="6D dynamic NVS: per-frame params, 100 frames at 1352x1014"),
    "c5": dict(kind="2d", H=2160, W=3840, N=3000000, blend="sum", shard="rows",
               desc="Scale sweep: 4K image, 3M 2D primitives, weighted sum, tile-row sharded"),
    "p3d": dict(kind="3d", H=256, W=256, N=20000, B=2, blend="alpha", scale_mult=4.0,
                desc="parity-only mini 3D"),
    "p6d": dict(kind="6d", H=96, W=128, N=5000, B=3, blend="alpha", scale_mult=4.0,
                desc="parity-only mini 6D"),
}


def make_config(name: str, seed: int = 0, **over) -> dict:
    """Build the full input set of a named config: dict(kind, H, W, B, N, blend,
    params, cams (3D), view_stride)."""
    c = dict(CONFIGS[name])
    c.update(over)
    kind, H, W, N = c["kind"], c["H"], c["W"], c["N"]
    if kind == "2d":
        p = gen2d(H, W, N, seed, cov_mode=c.get("cov_mode", "sigma"),
                  freq_std=c.get("freq_std", 0.5), phase=c.get("phase", False),
                  color_max=c.get("color_max", 0.1))
        return dict(c, B=1, params=p, cams=None, view_stride=0)
    B = c["B"]
    if kind == "3d":
        p = gen3d(N, seed, scale_mult=c.get("scale_mult", 1.0), sh_degree=c.get("sh_degree"))
        cams = ring_cameras(B, W, H)
        return dict(c, params=p, cams=cams, view_stride=0)
    p = gen6d(N, B, seed, scale_mult=c.get("scale_mult", 1.0), sh_degree=c.get("sh_degree"))
    cams = arc_cameras(B, W, H)
    return dict(c, params=p, cams=cams, view_stride=N)

"""Finite-difference pins of the oracle's analytic gradients (CPU only).

North-star check 'finite-difference gradients agree on tiny inputs' and
SPEC S:280 / S:289 / S:517: central differences in double precision of the
oracle's own forward (Eq. 3 / Eq. 4 with W') against
the analytic gradients for every parameter group ("explicit gradients for all
parameters"). Inputs are 16x16 images with <= 8 primitives and
every threshold margin >= 1e-3, so no FD step crosses a skip/clamp/stop.
"""
import math

import numpy as np
import pytest

from paper_2508_12615_b200 import gen

H = W = 16


def _loss(ora, cfg, p, dLdC, cams=None, vs=0):
    out = ora.forward(cfg, p, cams=cams, view_stride=vs)
    return float(np.sum(out["color"] * dLdC)), out


def _fd_check(ora, cfg, p, cams=None, vs=0, groups=None, h=1e-6, seed=0, min_margin=1e-3):
    rng = np.random.default_rng(seed)
    B = len(cams) if cams else 1
    dLdC = rng.uniform(-1, 1, (B * H * W, 3))
    L0, out0 = _loss(ora, cfg, p, dLdC, cams, vs)
    assert np.min(out0["margin"]) >= min_margin, np.min(out0["margin"])
    an = ora.forward_backward(cfg, p, dLdC, cams=cams, view_stride=vs)["grads"]
    groups = groups or list(an.keys())
    nchecked = 0
    for g in groups:
        if g not in p:
            continue
        arr = p[g]
        flat = arr.reshape(-1)
        ga = an[g].reshape(-1)
        for k in range(flat.size):
            old = flat[k]
            step = h * max(1.0, abs(old))
            flat[k] = old + step
            Lp, op = _loss(ora, cfg, p, dLdC, cams, vs)
            flat[k] = old - step
            Lm, om = _loss(ora, cfg, p, dLdC, cams, vs)
            flat[k] = old
            fd = (Lp - Lm) / (2 * step)
            err = abs(fd - ga[k])
            scale = max(abs(fd), abs(ga[k]))
            assert err <= 1e-4 * scale + 1e-7, (g, k, fd, ga[k])
            nchecked += 1
    return nchecked


def _p64(p):
    return {k: np.array(v, np.float64) for k, v in p.items()}


@pytest.mark.parametrize("mode", ["sigma", "cholesky", "rs"])
@pytest.mark.parametrize("blend", [False, True])
def test_fd_2d(ora, mode, blend):
    p = _p64(gen.gen2d(H, W, 6, seed=21, cov_mode=mode, freq_std=0.6, phase=True,
                       alpha=(0.3, 0.9), color_max=1.0, s0=2.5, depth=blend))
    cfg = ora.Cfg(width=W, height=H, cov2=mode, alpha_blend=blend, alpha_min=0.0,
                  alpha_max=0.99, T_min=0.0 if not blend else 1e-4)
    n = _fd_check(ora, cfg, p, min_margin=0.0 if not blend else 1e-3)
    assert n >= 6 * 12


@pytest.mark.parametrize("blend", [False, True])
def test_fd_2d_with_truncation(ora, blend):
    """Defaults (alpha_min = 1/255 skip, 0.99 clamp, 1e-4 stop) on margin-screened
    inputs: the derivative of the piecewise function (R25)."""
    for seed in range(30, 60):
        p = _p64(gen.gen2d(H, W, 6, seed=seed, cov_mode="cholesky", freq_std=0.5,
                           alpha=(0.3, 0.9), color_max=1.0, s0=2.5, depth=blend))
        cfg = ora.Cfg(width=W, height=H, cov2="cholesky", alpha_blend=blend)
        if np.min(ora.forward(cfg, p)["margin"]) >= 1e-3:
            break
    else:
        pytest.skip("no margin-screened seed")
    _fd_check(ora, cfg, p)


def _scene3d(n=6, seed=0, scale=0.12):
    rng = np.random.default_rng(seed)
    p = dict(mean=rng.normal(0, 0.35, (n, 3)), scale=rng.uniform(0.5, 1.5, (n, 3)) * scale,
             quat=rng.normal(size=(n, 4)), freq=rng.normal(0, 4.0, (n, 3)),
             phase=rng.uniform(-math.pi, math.pi, n), color=rng.uniform(0, 1, (n, 3)),
             opacity=rng.uniform(0.3, 0.9, n))
    return p


def _cams(B, seed=0):
    cams = []
    for v in range(B):
        a = 0.4 * v + 0.1 * seed
        R, t = gen.look_at((3 * math.sin(a), -0.4, -3 * math.cos(a)), (0, 0, 0))
        cams.append(dict(R=R, t=t, fx=40.0, fy=44.0, cx=8.0, cy=8.0, near=0.01, far=100.0))
    return cams


@pytest.mark.parametrize("blend", [False, True])
def test_fd_3d(ora, blend):
    """3-D chain (PAPER.md:106 Sigma = R S S^T R^T; :122 J W; :212 frequency
    transform): every partial pinned by FD, not by hand."""
    p = _scene3d(6, seed=3)
    cams = _cams(2)
    cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=blend, alpha_min=0.0,
                  dilation=0.3, T_min=1e-4 if blend else 0.0)
    _fd_check(ora, cfg, p, cams=cams, vs=0, min_margin=1e-3 if blend else 0.0)


def test_fd_3d_ewa_clamp_active(ora):
    """A primitive beyond 1.3x the half-FOV (clamped J) with a footprint reaching
    into the image: the clamp's zero partial matches FD (R6)."""
    p = _scene3d(3, seed=4, scale=0.3)
    p["mean"][0] = [2.3, 0.1, 0.0]
    p["scale"][0] = [0.9, 0.6, 0.7]
    cams = [dict(R=np.eye(3), t=np.array([0, 0, 3.0]), fx=20.0, fy=20.0, cx=8.0, cy=8.0,
                 near=0.01, far=100.0)]
    cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=False, alpha_min=0.0,
                  dilation=0.3)
    pr = ora.project3d(cfg, p, cams)
    x, y, z = p["mean"][0] + [0, 0, 3.0]
    assert abs(x / z) > 1.3 * W / (2 * 20.0)  # clamp active for primitive 0
    _fd_check(ora, cfg, p, cams=cams)


def test_fd_6d_per_frame_params(ora):
    """view_stride = N (per-frame parameters, Eq. 8): gradients land
    on each frame's own parameter rows."""
    n, B = 4, 2
    p = _scene3d(n * B, seed=5)
    cams = _cams(B, seed=1)
    cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=True, alpha_min=0.0,
                  dilation=0.3)
    _fd_check(ora, cfg, p, cams=cams, vs=n, groups=["mean", "scale", "quat", "freq", "opacity"])


def test_zero_residual_zero_gradient(ora):
    """dL/dC = 0 => all gradients exactly 0."""
    p = _p64(gen.gen2d(H, W, 8, seed=2))
    cfg = ora.Cfg(width=W, height=H)
    g = ora.forward_backward(cfg, p, np.zeros((H * W, 3)))["grads"]
    for v in g.values():
        assert np.all(v == 0.0)


def test_zero_freq_symmetric_residual(ora):
    """f = 0 and a residual symmetric about mu => dL/df = 0."""
    N = 16
    p = dict(mean=np.array([[8.0, 8.0]]), cov=np.array([[3.0, 0.5, 2.0]]),
             freq=np.zeros((1, 2)), color=np.array([[1.0, 0.5, 0.2]]), opacity=np.array([0.8]))
    rng = np.random.default_rng(0)
    r = rng.uniform(-1, 1, (N, N, 3))
    r = r + r[::-1, ::-1]  # point-symmetric about the image centre (8, 8)
    cfg = ora.Cfg(width=N, height=N)
    g = ora.forward_backward(cfg, p, r.reshape(-1, 3))["grads"]
    assert np.max(np.abs(g["freq"])) < 1e-12


def test_occluded_primitive_small_gradient(ora):
    """a primitive behind an (effective alpha 0.99) occluder gets
    gradients <= 1e-2 of its unoccluded ones."""
    rear = dict(mean=np.array([[8.0, 8.0]]), cov=np.array([[4.0, 0.0, 4.0]]),
                freq=np.array([[0.3, 0.2]]), color=np.array([[0.2, 0.9, 0.4]]),
                opacity=np.array([0.6]), depth=np.array([5.0]))
    front = dict(mean=np.array([[8.0, 8.0]]), cov=np.array([[400.0, 0.0, 400.0]]),
                 freq=np.array([[0.0, 0.0]]), color=np.array([[0.0, 0.0, 0.0]]),
                 opacity=np.array([1.0]), depth=np.array([1.0]))
    both = {k: np.concatenate([rear[k], front[k]]) for k in rear}
    cfg = ora.Cfg(width=16, height=16, alpha_blend=True, T_min=0.0)
    rng = np.random.default_rng(1)
    dL = rng.uniform(-1, 1, (256, 3))
    g1 = ora.forward_backward(cfg, rear, dL)["grads"]
    g2 = ora.forward_backward(cfg, both, dL)["grads"]
    for k in ("mean", "cov", "freq", "color", "opacity"):
        assert np.max(np.abs(g2[k][0])) <= 1.5e-2 * np.max(np.abs(g1[k][0])) + 1e-12, k


@pytest.mark.parametrize("blend", [False, True])
def test_fd_3d_exact_projection(ora, blend):
    """NEXT-1 exact z-integration (beta = exp(-1/2 f_z^2 v)): the
    oracle's exact-mode gradients (Jacobian of its pinned exact projection)
    agree with central FD of the whole exact-mode pipeline."""
    p = _scene3d(5, seed=8)
    p["freq"] = p["freq"] * 2.0   # make f_hat_z (and beta < 1) matter
    cams = _cams(2, seed=2)
    cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=blend, alpha_min=0.0,
                  dilation=0.3, exact_proj=True, T_min=1e-4 if blend else 0.0)
    pr = ora.project3d(cfg, p, cams)
    beta = pr.field("beta")[pr.flag == 0]
    assert beta.min() < 0.9  # the exact mode differs from the paper mode here
    _fd_check(ora, cfg, p, cams=cams, min_margin=1e-3 if blend else 0.0, h=1e-6)


def test_exact_chain_matches_paper_chain_when_fz_zero(ora):
    """With f = 0, exact and paper modes coincide (beta = 1, f' = 0): the
    FD-Jacobian exact chain must reproduce the hand-derived paper chain."""
    p = _scene3d(5, seed=9)
    p["freq"] = np.zeros_like(p["freq"])
    cams = _cams(2, seed=3)
    rng = np.random.default_rng(0)
    dL = rng.uniform(-1, 1, (2 * H * W, 3))
    ce = ora.Cfg(width=W, height=H, prim3d=True, alpha_min=0.0, dilation=0.3, exact_proj=True)
    cp = ora.Cfg(width=W, height=H, prim3d=True, alpha_min=0.0, dilation=0.3)
    ge = ora.forward_backward(ce, p, dL, cams=cams)["grads"]
    gpp = ora.forward_backward(cp, p, dL, cams=cams)["grads"]
    for k in ("mean", "scale", "quat", "opacity", "color"):
        np.testing.assert_allclose(ge[k], gpp[k], rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("blend", [False, True])
def test_fd_3d_sh(ora, blend):
    """NEXT-3 SH colour: dL/dsh and the view-direction term of
    dL/dmu against central FD of the whole pipeline (degree 3, two views)."""
    p = _scene3d(5, seed=11)
    del p["color"]
    rng = np.random.default_rng(12)
    p["sh"] = rng.normal(0, 0.3, (5, 16, 3))
    p["sh"][:, 0, :] = rng.uniform(0.5, 1.5, (5, 3))  # colours well above the clamp
    cams = _cams(2, seed=4)
    cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=blend, alpha_min=0.0,
                  dilation=0.3, T_min=1e-4 if blend else 0.0, sh_degree=3)
    n = _fd_check(ora, cfg, p, cams=cams, groups=["sh", "mean"],
                  min_margin=1e-3 if blend else 0.0)
    assert n == 5 * 48 + 15

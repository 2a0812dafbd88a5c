"""Pins of the oracle's spherical-harmonic colour (NEXT-3; PAPER.md:106,
settings of 3DGS P:380). CPU only.

The basis is pinned by properties a wrong constant, sign-free typo or
swapped component would break: orthonormality on the sphere (Gauss-Legendre x
uniform quadrature, exact for these polynomial degrees), the addition theorem
sum_m Y_lm(d)^2 = (2l+1)/(4 pi) at every direction, and parity
Y_lm(-d) = (-1)^l Y_lm(d). The colour path is pinned by the degree-0 closed
form and, for gradients, by finite differences of the whole pipeline
(test_oracle_grad.py::test_fd_3d_sh).
"""
import math

import numpy as np
import pytest


def _sphere_quadrature(nt=24, nphi=48):
    x, w = np.polynomial.legendre.leggauss(nt)  # cos(theta)
    phi = (np.arange(nphi) + 0.5) * 2 * math.pi / nphi
    ct, ph = np.meshgrid(x, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    d = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    wt = (w[:, None] * np.full(nphi, 2 * math.pi / nphi)[None, :]).reshape(-1)
    return d, wt


def test_sh_orthonormal(ora):
    d, w = _sphere_quadrature()
    Y = ora.sh_basis(3, d)
    G = (Y * w[:, None]).T @ Y
    np.testing.assert_allclose(G, np.eye(16), atol=1e-12)


def test_sh_addition_theorem_and_parity(ora):
    rng = np.random.default_rng(0)
    d = rng.normal(size=(200, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    Y = ora.sh_basis(3, d)
    Yn = ora.sh_basis(3, -d)
    for l in range(4):
        sl = slice(l * l, (l + 1) * (l + 1))
        np.testing.assert_allclose((Y[:, sl] ** 2).sum(1), (2 * l + 1) / (4 * math.pi),
                                   rtol=1e-12)
        np.testing.assert_allclose(Yn[:, sl], (-1) ** l * Y[:, sl], atol=1e-14)
    # lower degrees are prefixes of the degree-3 basis
    np.testing.assert_array_equal(ora.sh_basis(1, d), Y[:, :4])


def test_sh_degree0_colour_closed_form(ora):
    cams = [dict(R=np.eye(3), t=np.array([0.0, 0.0, 3.0]), fx=10.0, fy=10.0, cx=8.0, cy=8.0,
                 near=0.01, far=100.0)]
    mean = np.array([[0.1, -0.2, 0.3], [0.0, 0.0, 0.0]])
    sh = np.array([[[1.0, -0.5, -3.0]], [[0.0, 0.2, 0.4]]])
    rgb = ora.sh_colors(0, mean, sh, cams, 2)
    c0 = 1.0 / (2.0 * math.sqrt(math.pi))
    np.testing.assert_allclose(rgb, np.maximum(0.0, c0 * sh[:, 0, :] + 0.5), rtol=1e-15)
    assert rgb[0, 2] == 0.0  # clamped


def test_sh_colour_depends_on_view_direction_only(ora):
    """Moving the primitive along the viewing ray leaves its colour unchanged;
    the camera centre C = -R^T t enters through d = (mu - C)/|mu - C|."""
    rng = np.random.default_rng(3)
    R, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    t = rng.normal(size=3)
    C = -R.T @ t
    cams = [dict(R=R, t=t, fx=10.0, fy=10.0, cx=8.0, cy=8.0, near=0.01, far=100.0)]
    mu = C + np.array([0.3, -0.4, 1.2])
    sh = rng.normal(0, 0.3, (1, 16, 3))
    a = ora.sh_colors(3, mu[None], sh, cams, 1)
    b = ora.sh_colors(3, (C + 2.5 * (mu - C))[None], sh, cams, 1)
    np.testing.assert_allclose(a, b, rtol=1e-12)

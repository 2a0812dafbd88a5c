"""Pins of the oracle's NEXT-2 fitting-step functions (CPU only).

Each check is a closed form or a SPEC example, not a retyping of the formula:
SPEC S:336-344 (train_step), S:345-352 (evaluate), S:321-324 (AdamState),
S:422-427 (zone plate), S:328-331 (init_primitives).
"""
import math

import numpy as np

from paper_2508_12615_b200 import gen


def test_loss_closed_forms(ora):
    # mid-gray vs black: MSE 0.25 -> PSNR 6.02 dB
    img = np.full((1, 3, 8, 8), 0.5)
    loss, g = ora.loss_l2(img, np.zeros_like(img))
    assert loss == 0.25
    assert abs(10 * math.log10(1 / loss) - 6.0206) < 1e-4
    # constant offset c: loss c^2, gradient 2c/n everywhere
    rng = np.random.default_rng(0)
    t = rng.uniform(0, 1, (1, 3, 5, 7))
    loss, g = ora.loss_l2(t + 0.1, t)
    assert abs(loss - 0.01) < 1e-15
    assert np.allclose(g, 0.2 / t.size, rtol=1e-12, atol=0)


def test_loss_gradient_by_finite_differences(ora):
    rng = np.random.default_rng(1)
    a, b = rng.uniform(0, 1, (3, 4, 4)), rng.uniform(0, 1, (3, 4, 4))
    _, g = ora.loss_l2(a, b)
    h = 1e-6
    for idx in [(0, 0, 0), (1, 2, 3), (2, 3, 1)]:
        ap, am = a.copy(), a.copy()
        ap[idx] += h
        am[idx] -= h
        fd = (ora.loss_l2(ap, b)[0] - ora.loss_l2(am, b)[0]) / (2 * h)
        assert abs(fd - g[idx]) < 1e-9


def test_adam_first_step_is_signed_lr(ora):
    """t = 1: m_hat = g, v_hat = g^2 -> update = -lr g / (|g| + eps) = -lr sign(g)."""
    rng = np.random.default_rng(2)
    p0 = rng.normal(size=100)
    g = rng.normal(size=100)
    p, m, v, _ = ora.adam_step(p0, g, np.zeros(100), np.zeros(100), 1, lr=0.01)
    assert np.allclose(p, p0 - 0.01 * np.sign(g), rtol=0, atol=1e-14)
    assert np.allclose(m, 0.1 * g) and np.allclose(v, 0.001 * g * g)


def test_adam_constant_gradient_moves_lr_per_step(ora):
    """Bias correction makes m_hat = g and v_hat = g^2 at every t for a constant
    gradient, so the parameter moves exactly lr per step."""
    p = np.array([1.0, -2.0, 0.5])
    g = np.array([0.3, -1e-3, 7.0])
    m = np.zeros(3)
    v = np.zeros(3)
    for t in range(1, 11):
        p, m, v, _ = ora.adam_step(p, g, m, v, t, lr=0.05)
    assert np.allclose(p, np.array([1.0, -2.0, 0.5]) - 10 * 0.05 * np.sign(g), atol=1e-12)


def test_adam_zero_residual_leaves_parameters(ora):
    """zero gradient -> parameters unchanged (<= 1e-10)."""
    p0 = np.array([0.3, 4.0])
    p, m, v, _ = ora.adam_step(p0, np.zeros(2), np.zeros(2), np.zeros(2), 1, lr=1.0)
    assert np.max(np.abs(p - p0)) <= 1e-10


def test_adam_sigmoid_chain(ora):
    """act = sigmoid(theta), dL/dtheta = dL/dact * s (1 - s): at theta = 0 the
    derivative is 1/4 (the chained first moment is (1 - b1) g / 4)."""
    p, m, v, act = ora.adam_step(np.zeros(2), np.array([2.0, -4.0]), np.zeros(2), np.zeros(2),
                                 1, lr=0.1, activation="sigmoid")
    assert np.allclose(m, 0.1 * np.array([0.5, -1.0]))
    assert np.allclose(p, [-0.1, 0.1])
    assert np.allclose(act, 1 / (1 + np.exp(-p)))
    h = 1e-6
    s = ora.sigmoid
    assert abs((s(0.3 + h) - s(0.3 - h)) / (2 * h) - s(0.3) * (1 - s(0.3))) < 1e-10


def test_zone_plate_examples():
    z = gen.zone_plate(33, 33, k=40.0)
    assert z.shape == (3, 33, 33)
    assert abs(z[0, 16, 16] - 0.5) < 1e-3  # centre pixel, u = v ~ 0
    assert np.all(z >= 0) and np.all(z <= 1)
    assert np.allclose(gen.zone_plate(32, 32, k=0.0), 0.5)
    # local DFT peak frequency grows outwards (chirp)
    z = gen.zone_plate(256, 256, k=200.0)[0]

    def peak(patch):
        F = np.abs(np.fft.fft2(patch - patch.mean()))
        fy, fx = np.unravel_index(np.argmax(F), F.shape)
        fy, fx = min(fy, 32 - fy), min(fx, 32 - fx)
        return math.hypot(fx, fy)
    assert peak(z[:32, :32]) > peak(z[112:144, 112:144])


def test_init_from_target():
    t = np.full((3, 16, 16), 0.25, np.float32)
    p = gen.init2d_from_target(t, 1, seed=0)
    assert np.allclose(p["color"], 0.25)  # constant image: colour is the constant
    p = gen.init2d_from_target(gen.smooth_target(32, 48, seed=1), 64, seed=3)
    q = gen.init2d_from_target(gen.smooth_target(32, 48, seed=1), 64, seed=3)
    assert all(np.array_equal(p[k], q[k]) for k in p)  # seeded -> bit-identical
    s = math.sqrt(32 * 48 / 64)
    assert np.allclose(p["cov"], [s, 0, s]) and np.all(p["opacity"] == 0)
    assert p["mean"][:, 0].max() < 48 and p["mean"][:, 1].max() < 32

"""Pins of the oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it checks. Nothing here compares the oracle with
itself: values come from closed forms, SPEC/paper worked examples
(tests/golden/spec_examples.json), independent library routes (numpy linalg,
scipy rotations, numpy FFT, numerical quadrature) or brute force.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_2508_12615_b200 import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def conic_of(cov):
    """inverse of [[sxx, sxy],[sxy, syy]] via numpy (independent route)."""
    S = np.array([[cov[0], cov[1]], [cov[1], cov[2]]], np.float64)
    A = np.linalg.inv(S)
    return [A[0, 0], A[0, 1], A[1, 1]]


# ---------------------------------------------------------------- Eq. 1 / Eq. 6
@pytest.mark.parametrize("ex", GOLD["eval_gaussian"])
def test_gaussian_golden(ora, ex):
    """Gaussian closed forms (Eq. 1)."""
    v = ora.eval_gaussian2(conic_of(ex["cov"]), *ex["d"])
    assert v == pytest.approx(ex["value"], abs=1e-15)


@pytest.mark.parametrize("ex", GOLD["eval_wavelet"])
def test_wavelet_golden(ora, ex):
    """centre value and cosine zero crossing (Eq. 6)."""
    v = ora.eval_wavelet2(conic_of(ex["cov"]), ex["f"], 0.0, ex["beta"], *ex["d"])
    assert v == pytest.approx(ex["value"], abs=1e-15)


def test_zero_frequency_is_gaussian_bitwise(ora):
    """'the Gaussian primitive can be considered a subset ... by
    setting f to 0': with f = 0 and phi = 0, W == G bit for bit (h = 1 exactly)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        cov = [rng.uniform(0.5, 4), rng.uniform(-0.3, 0.3), rng.uniform(0.5, 4)]
        A = conic_of(cov)
        dx, dy = rng.normal(0, 2, 2)
        assert ora.eval_wavelet2(A, [0.0, 0.0], 0.0, 1.0, dx, dy) == ora.eval_gaussian2(A, dx, dy)
        # and G equals exp(-1/2 d^T Sigma^{-1} d) via a linear solve
        S = np.array([[cov[0], cov[1]], [cov[1], cov[2]]])
        d = np.array([dx, dy])
        ref = math.exp(-0.5 * d @ np.linalg.solve(S, d))
        assert ora.eval_gaussian2(A, dx, dy) == pytest.approx(ref, rel=1e-12)


def test_centre_value_amplitude_cos_phase(ora):
    """North-star check 'value at the primitive centre equals amplitude*cos(phase)':
    W(mu) = 1/2 (1 + beta cos phi)  <=>  2 W(mu) - 1 = beta cos phi (R1)."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        beta, phi = rng.uniform(0, 1), rng.uniform(-math.pi, math.pi)
        v = ora.eval_wavelet2([1, 0, 1], [0.3, 0.2], phi, beta, 0.0, 0.0)
        assert 2 * v - 1 == pytest.approx(beta * math.cos(phi), abs=1e-15)


def test_envelope_bound_and_symmetry(ora):
    """0 <= W <= G <= 1 and W(mu+d) = W(mu-d) (phi = 0)."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        cov = [rng.uniform(0.5, 4), rng.uniform(-0.3, 0.3), rng.uniform(0.5, 4)]
        A = conic_of(cov)
        f = rng.normal(0, 1.5, 2)
        d = rng.normal(0, 3, 2)
        w = ora.eval_wavelet2(A, f, 0.0, 1.0, *d)
        g = ora.eval_gaussian2(A, *d)
        assert 0.0 <= w <= g <= 1.0
        assert w == pytest.approx(ora.eval_wavelet2(A, f, 0.0, 1.0, *(-d)), abs=1e-15)


# ------------------------------------------------ covariance constructions
@pytest.mark.parametrize("ex", GOLD["cov_cholesky"])
def test_cholesky_golden(ora, ex):
    """SPEC S:105-107 (PAPER.md:299 'Cholesky')."""
    np.testing.assert_allclose(ora.cov2d("cholesky", ex["l"]), ex["sigma"], atol=1e-15)


@pytest.mark.parametrize("ex", GOLD["cov_rs"])
def test_rs_golden(ora, ex):
    """SPEC S:114-115 (PAPER.md:299 'RS'; Sigma = R S S^T R^T)."""
    np.testing.assert_allclose(ora.cov2d("rs", ex["p"]), ex["sigma"], atol=1e-14)


def test_cov_params_match_matrix_products(ora):
    """Cholesky = L L^T and RS = R diag(s^2) R^T computed with numpy matmul, and
    RS periodicity Sigma(theta) = Sigma(theta + pi)."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        l1, l2, l3 = rng.normal(size=3)
        L = np.array([[l1, 0], [l2, l3]])
        S = L @ L.T
        np.testing.assert_allclose(ora.cov2d("cholesky", [l1, l2, l3]),
                                   [S[0, 0], S[0, 1], S[1, 1]], rtol=1e-13, atol=1e-14)
        th, sx, sy = rng.uniform(-4, 4), rng.uniform(0.1, 3), rng.uniform(0.1, 3)
        R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
        S = R @ np.diag([sx * sx, sy * sy]) @ R.T
        got = ora.cov2d("rs", [th, sx, sy])
        np.testing.assert_allclose(got, [S[0, 0], S[0, 1], S[1, 1]], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(ora.cov2d("rs", [th + math.pi, sx, sy]), got, atol=1e-12)


# ------------------------------------------------------------- projection
def _cam_identity(W=64, H=64, f=1.0):
    return dict(R=np.eye(3), t=np.zeros(3), fx=f, fy=f, cx=0.0, cy=0.0, near=0.01, far=100.0)


def _one3d(mu, scale=(1, 1, 1), quat=(1, 0, 0, 0), freq=(0, 0, 0), alpha=1.0):
    return dict(mean=np.array([mu], np.float64), scale=np.array([scale], np.float64),
                quat=np.array([quat], np.float64), freq=np.array([freq], np.float64),
                color=np.array([[1, 1, 1]], np.float64), opacity=np.array([alpha], np.float64))


@pytest.mark.parametrize("ex", GOLD["projection"])
def test_projection_golden(ora, ex):
    """J, Sigma' and f_hat closed forms
    (PAPER.md:122 Sigma_hat = J W Sigma W^T J^T; PAPER.md:212 frequency)."""
    cfg = ora.Cfg(width=64, height=64, prim3d=True, alpha_blend=True,
                  dilation=ex.get("dilation", 0.0), ewa_clamp=False)
    p = _one3d(ex["mu"], scale=ex.get("scale", (1, 1, 1)), freq=ex.get("freq", (0, 0, 0)))
    pr = ora.project3d(cfg, p, [_cam_identity()])
    assert pr.flag[0] in (0, 4)
    if "sigma_prime" in ex:
        got = [pr.field("sxx")[0], pr.field("sxy")[0], pr.field("syy")[0]]
        np.testing.assert_allclose(got, ex["sigma_prime"], atol=1e-14)
    if "f_prime" in ex:
        np.testing.assert_allclose([pr.field("fx")[0], pr.field("fy")[0]], ex["f_prime"],
                                   atol=1e-14)


def _ray_integral_profile(p, cam, pixels, zlo, zhi, nz=4001):
    """Brute-force line integral of the 3-D wavelet (Eq. 6 in world space) along
    the camera ray of each pixel, parameterised by camera depth z (ray space
    coordinate 3 = z). Independent of the oracle's projection: the
    3-D covariance is built with scipy's rotation from the quaternion."""
    from scipy.spatial.transform import Rotation
    w, x, y, z = p["quat"][0]
    Rq = Rotation.from_quat([x, y, z, w]).as_matrix()
    S3 = Rq @ np.diag(np.asarray(p["scale"][0]) ** 2) @ Rq.T
    Si = np.linalg.inv(S3)
    R, t = np.asarray(cam["R"], np.float64), np.asarray(cam["t"], np.float64)
    mu = np.asarray(p["mean"][0], np.float64)
    f = np.asarray(p["freq"][0], np.float64)
    zs = np.linspace(zlo, zhi, nz)
    out = []
    for (u, v) in pixels:
        xc = np.stack([(u - cam["cx"]) / cam["fx"] * zs, (v - cam["cy"]) / cam["fy"] * zs, zs], 1)
        xw = (xc - t) @ R  # R^T (x_c - t)
        d = xw - mu
        q = np.einsum("ni,ij,nj->n", d, Si, d)
        val = np.exp(-0.5 * q) * 0.5 * (1 + np.cos(d @ f))
        out.append(np.trapezoid(val, zs))
    return np.array(out)


@pytest.mark.parametrize("exact", [False, True])
def test_projection_matches_ray_integral(ora, exact):
    """Eq. 2 / Eq. 7 and the frequency transform
    (PAPER.md:212): the projected 2-D wavelet W'(x') must equal the z-integral
    of the 3-D wavelet along each pixel's ray, up to the local-affine (EWA)
    approximation error O(sigma/z). Exact mode matches for any f; paper mode
    (beta = 1, f' = f_hat_xy) only when f_hat_z = 0 and there are no x-z / y-z
    cross terms, i.e. the in-plane frequency case used here for exact=False."""
    rng = np.random.default_rng(5 + exact)
    W = H = 64
    f_px = 400.0
    cam = dict(R=gen.look_at((0.3, -0.2, -5.0), (0.05, 0.02, 0.0))[0],
               t=gen.look_at((0.3, -0.2, -5.0), (0.05, 0.02, 0.0))[1],
               fx=f_px, fy=f_px * 1.1, cx=W / 2, cy=H / 2, near=0.01, far=100.0)
    for trial in range(3):
        mu = rng.normal(0, 0.05, 3)
        scale = rng.uniform(0.01, 0.03, 3)
        q = rng.normal(size=4)
        if exact:
            freq = rng.normal(0, 60.0, 3)
        else:
            # isotropic envelope => Sigma_hat has no cross terms after the
            # affine map only approximately; use scale iso + f orthogonal to the
            # viewing ray so f_hat_z ~ 0.
            scale = np.full(3, 0.02)
            R = np.asarray(cam["R"], np.float64)
            fc = np.array([rng.normal(0, 60), rng.normal(0, 60), 0.0])
            freq = R.T @ fc
        p = _one3d(mu, scale, q, freq)
        cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=True, ewa_clamp=False,
                      exact_proj=exact, alpha_min=0.0, dilation=0.0)
        pr = ora.project3d(cfg, p, [cam])
        r = pr.rec[0]
        mux, muy = r[0], r[1]
        pix = [(mux + dx, muy + dy) for dx in np.linspace(-6, 6, 7) for dy in np.linspace(-6, 6, 7)]
        zc = (np.asarray(cam["R"]) @ mu + np.asarray(cam["t"]))[2]
        ray = _ray_integral_profile(p, cam, pix + [(mux, muy)], zc - 0.3, zc + 0.3)
        ray = ray[:-1] / ray[-1] * (0.5 * (1 + r[8]))  # normalise to the kernel's centre value
        A = [r[2], r[3], r[4]]
        ker = np.array([ora.eval_wavelet2(A, [r[5], r[6]], 0.0, r[8], u - mux, v - muy)
                        for (u, v) in pix])
        assert np.max(np.abs(ray - ker)) < 5e-3, (trial, np.max(np.abs(ray - ker)))


def test_phase_invariance_contravariant(ora):
    """DESIGN.md R3: with f' = (J3 W)^{-T} f the phase is invariant under the
    local affine map: f'.(M d) = f.d for the in-plane components when the
    depth offset is zero. Checked against numpy's inverse of J3 R."""
    rng = np.random.default_rng(6)
    W = H = 128
    for _ in range(20):
        R, t = gen.look_at(rng.normal(0, 1, 3) + np.array([0, 0, -6]), (0, 0, 0))
        cam = dict(R=R, t=t, fx=300.0, fy=280.0, cx=64.0, cy=64.0, near=0.01, far=100.0)
        mu = rng.normal(0, 0.3, 3)
        f = rng.normal(0, 5, 3)
        p = _one3d(mu, freq=f)
        cfg = ora.Cfg(width=W, height=H, prim3d=True, alpha_blend=True, ewa_clamp=False)
        pr = ora.project3d(cfg, p, [cam])
        x, y, z = R @ mu + t
        J3 = np.array([[300 / z, 0, -300 * x / z ** 2], [0, 280 / z, -280 * y / z ** 2], [0, 0, 1]])
        fhat = np.linalg.inv(J3 @ R).T @ f
        np.testing.assert_allclose([pr.rec[0][5], pr.rec[0][6]], fhat[:2], rtol=1e-10, atol=1e-12)
        d = rng.normal(0, 0.1, 3)
        assert fhat @ (J3 @ R @ d) == pytest.approx(f @ d, rel=1e-9, abs=1e-12)


def test_frustum_clamp_and_cull(ora):
    """Q6/Q15 readings: behind-camera primitives cull with flag 1; far off-axis
    primitives get the clamped J (finite, smaller footprint than unclamped)."""
    cam = dict(R=np.eye(3), t=np.zeros(3), fx=100.0, fy=100.0, cx=32.0, cy=32.0, near=0.01,
               far=100.0)
    cfg = ora.Cfg(width=64, height=64, prim3d=True, alpha_blend=True, dilation=0.3)
    pr = ora.project3d(cfg, _one3d((0, 0, -1.0)), [cam])
    assert pr.flag[0] == 1 and pr.count[0] == 0
    pr = ora.project3d(cfg, _one3d((0, 0, 200.0)), [cam])
    assert pr.flag[0] == 1
    pc = ora.project3d(cfg, _one3d((5.0, 0, 1.0), scale=(0.2, 0.2, 0.2)), [cam])
    cfg2 = ora.Cfg(width=64, height=64, prim3d=True, alpha_blend=True, dilation=0.3,
                   ewa_clamp=False)
    pu = ora.project3d(cfg2, _one3d((5.0, 0, 1.0), scale=(0.2, 0.2, 0.2)), [cam])
    assert pc.field("sxx")[0] < pu.field("sxx")[0]


# ---------------------------------------------------------------- rendering
def _prims2d(mu, cov, f=(0, 0), c=(1, 0, 0), a=1.0, phase=None):
    p = dict(mean=np.array([mu], np.float64), cov=np.array([cov], np.float64),
             freq=np.array([f], np.float64), color=np.array([c], np.float64),
             opacity=np.array([a], np.float64))
    if phase is not None:
        p["phase"] = np.array([phase], np.float64)
    return p


def test_render_sum_golden_single(ora):
    """one primitive, pixel at mu, c = (1,0,0), alpha = 0.5 -> (0.5,0,0)
    (Eq. 4)."""
    cfg = ora.Cfg(width=16, height=16)
    out = ora.forward(cfg, _prims2d((8.5, 4.5), (2, 0.3, 1.5), f=(0.4, 0.9), a=0.5),
                      pix=[4 * 16 + 8])
    np.testing.assert_allclose(out["color"][0], [0.5, 0, 0], atol=1e-15)


def test_render_centre_amplitude_cos_phase(ora):
    """North-star 'value at the centre equals amplitude*cos(phase)': one
    primitive centred on a pixel centre, alpha = c = 1: 2 C(mu) - 1 = cos(phi)."""
    rng = np.random.default_rng(7)
    cfg = ora.Cfg(width=16, height=16, alpha_min=0.0)
    for _ in range(20):
        phi = rng.uniform(-math.pi, math.pi)
        out = ora.forward(cfg, _prims2d((3.5, 9.5), (3, 0.2, 2), f=rng.normal(0, 1, 2),
                                        c=(1, 1, 1), a=1.0, phase=phi), pix=[9 * 16 + 3])
        assert 2 * out["color"][0, 0] - 1 == pytest.approx(math.cos(phi), abs=1e-14)


def test_render_empty_and_linearity(ora):
    """empty scene renders 0; SUM mode is linear in the set of
    primitives (Eq. 4 is a sum), checked to 1e-12."""
    cfg = ora.Cfg(width=32, height=24)
    p = gen.gen2d(24, 32, 40, seed=3, freq_std=0.6)
    pd = {k: v.astype(np.float64) for k, v in p.items()}
    full = ora.forward(cfg, pd)["color"]
    A = {k: v[:17] for k, v in pd.items()}
    Bp = {k: v[17:] for k, v in pd.items()}
    sA = ora.forward(cfg, A)["color"]
    sB = ora.forward(cfg, Bp)["color"]
    np.testing.assert_allclose(full, sA + sB, atol=1e-12)
    empty = {k: v[:0] for k, v in pd.items()}
    assert np.all(ora.forward(cfg, empty)["color"] == 0.0)


def test_render_sum_bruteforce_definition(ora):
    """Eq. 4 with W' written as a numpy sum over all
    primitives with explicit inverses (alpha_min = 0: no truncation, the plain
    definition)."""
    H, W = 12, 10
    cfg = ora.Cfg(width=W, height=H, alpha_min=0.0, cov2="rs")
    p = gen.gen2d(H, W, 9, seed=5, cov_mode="rs", freq_std=0.8, phase=True, alpha=(0.2, 1.0))
    pd = {k: v.astype(np.float64) for k, v in p.items()}
    got = ora.forward(cfg, pd)["color"].reshape(H, W, 3)
    ys, xs = np.mgrid[0:H, 0:W] + 0.5
    ref = np.zeros((H, W, 3))
    for i in range(9):
        th, sx, sy = pd["cov"][i]
        R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
        Si = np.linalg.inv(R @ np.diag([sx * sx, sy * sy]) @ R.T)
        d = np.stack([xs - pd["mean"][i, 0], ys - pd["mean"][i, 1]], -1)
        q = np.einsum("hwi,ij,hwj->hw", d, Si, d)
        Wk = 0.5 * (np.cos(d @ pd["freq"][i] + pd["phase"][i]) + 1) * np.exp(-0.5 * q)
        ref += pd["opacity"][i] * Wk[..., None] * pd["color"][i]
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-13)


def test_render_gaussian_subset(ora):
    """SPEC S:292 / PAPER.md:191: all f = 0 => the render equals a carrier-free
    Gaussian-only brute force (Eq. 4 with G')."""
    H, W = 16, 16
    cfg = ora.Cfg(width=W, height=H)
    p = gen.gen2d(H, W, 12, seed=8, freq_std=0.0)
    pd = {k: v.astype(np.float64) for k, v in p.items()}
    got = ora.forward(cfg, pd)["color"].reshape(H, W, 3)
    ys, xs = np.mgrid[0:H, 0:W] + 0.5
    ref = np.zeros((H, W, 3))
    for i in range(12):
        sxx, sxy, syy = pd["cov"][i]
        Si = np.linalg.inv(np.array([[sxx, sxy], [sxy, syy]]))
        d = np.stack([xs - pd["mean"][i, 0], ys - pd["mean"][i, 1]], -1)
        g = pd["opacity"][i] * np.exp(-0.5 * np.einsum("hwi,ij,hwj->hw", d, Si, d))
        ref += np.where(g >= cfg.alpha_min, g, 0.0)[..., None] * pd["color"][i]
    np.testing.assert_allclose(got, ref, atol=1e-14)


def test_alpha_golden_and_occlusion(ora):
    """SPEC S:269 (alpha = 1 at centre -> 0.99 c) and S:270 (front a = 0.99 =>
    rear contributes <= 0.01 c) — Eq. 3, PAPER.md:125-129 with the 0.99 clamp."""
    cfg = ora.Cfg(width=16, height=16, alpha_blend=True, alpha_max=0.99)
    p = _prims2d((8.5, 8.5), (4, 0, 4), c=(0.2, 0.4, 0.8), a=1.0)
    p["depth"] = np.array([1.0])
    out = ora.forward(cfg, p, pix=[8 * 16 + 8])
    np.testing.assert_allclose(out["color"][0], GOLD["render_alpha"][0]["pixel"], atol=1e-12)
    # two primitives: front opaque, rear white
    p2 = {k: np.concatenate([v, v]) for k, v in p.items()}
    p2["color"] = np.array([[0, 0, 0], [1, 1, 1]], np.float64)
    p2["depth"] = np.array([1.0, 2.0])
    out = ora.forward(cfg, p2, pix=[8 * 16 + 8])
    assert np.all(out["color"][0] <= 0.01 + 1e-15)


def _composite_product_form(ws, cs, bg):
    """Eq. 3 literally: C = sum_i c_i a_i prod_{j<i} (1 - a_j) + bg prod (1 - a_j)."""
    C = np.zeros(3)
    for i in range(len(ws)):
        C += cs[i] * ws[i] * np.prod([1 - ws[j] for j in range(i)])
    return C + bg * np.prod([1 - w for w in ws])


def test_alpha_bruteforce_product_form(ora):
    """brute-force <= 5 primitive compositor in product form of
    Eq. 3, depth-ordered, no truncation (alpha_min = 0,
    alpha_max = 1, T_min = 0). Also convex hull and transmittance monotonicity."""
    rng = np.random.default_rng(9)
    H, W = 8, 8
    bg = np.array([0.1, 0.2, 0.3])
    cfg = ora.Cfg(width=W, height=H, alpha_blend=True, alpha_min=0.0, alpha_max=1.0, T_min=0.0,
                  bg=tuple(bg))
    for trial in range(20):
        n = rng.integers(1, 6)
        p = gen.gen2d(H, W, int(n), seed=100 + trial, freq_std=0.7, alpha=(0.1, 0.95),
                      depth=True, color_max=1.0)
        pd = {k: v.astype(np.float64) for k, v in p.items()}
        out = ora.forward(cfg, pd)
        order = np.argsort(pd["depth"], kind="stable")
        for pix in range(H * W):
            y, x = divmod(pix, W)
            ws, cs = [], []
            for i in order:
                sxx, sxy, syy = pd["cov"][i]
                Si = np.linalg.inv(np.array([[sxx, sxy], [sxy, syy]]))
                d = np.array([x + 0.5, y + 0.5]) - pd["mean"][i]
                Wk = 0.5 * (1 + math.cos(d @ pd["freq"][i])) * math.exp(-0.5 * d @ Si @ d)
                ws.append(pd["opacity"][i] * Wk)
                cs.append(pd["color"][i])
            ref = _composite_product_form(ws, cs, bg)
            np.testing.assert_allclose(out["color"][pix], ref, rtol=1e-12, atol=1e-14)
            # convex hull of {bg} U {c_i}: each channel within [min, max]
            allc = np.vstack(cs + [bg])
            assert np.all(out["color"][pix] >= allc.min(0) - 1e-12)
            assert np.all(out["color"][pix] <= allc.max(0) + 1e-12)
            assert 0.0 <= out["T"][pix] <= 1.0


def test_alpha_early_stop_rule(ora):
    """DESIGN.md R10 (T_min stop; crossing entry not composited): a front
    primitive leaving T = 1e-3, then one with a = 0.95 (T' = 5e-5 < 1e-4): the
    second is skipped entirely."""
    cfg = ora.Cfg(width=4, height=4, alpha_blend=True, alpha_max=0.999)
    p = dict(mean=np.array([[2.5, 2.5], [2.5, 2.5]]), cov=np.array([[50, 0, 50], [50, 0, 50]]),
             freq=np.zeros((2, 2)), color=np.array([[1, 0, 0], [0, 1, 0]], np.float64),
             opacity=np.array([0.999, 0.95]), depth=np.array([1.0, 2.0]))
    out = ora.forward(cfg, p, pix=[2 * 4 + 2])
    np.testing.assert_allclose(out["color"][0], [0.999, 0, 0], atol=1e-12)
    assert out["T"][0] == pytest.approx(1e-3, rel=1e-9)
    assert out["ncomp"][0] == 1


# --------------------------------------------------------------- spectrum
def test_fft_peak_at_frequency(ora):
    """PAPER.md:259-262 (Sec. 4.2): modulation shifts the envelope's spectrum to
    +-f. 256^2 SUM render of one primitive (sigma = 4 px, f = (2.0, -1.5) rad/px):
    the non-DC |DFT| peak (DC disc of radius 3N/(2 pi sigma) bins excluded) is
    within 1 bin of +-f N/(2 pi); |DFT| matches the analytic spectrum
    1/2 G^(w) + 1/4 [G^(w-f) + G^(w+f)] within 2% at the top-3 bins."""
    N = 256
    sig = 4.0
    f = np.array([2.0, -1.5])
    cfg = ora.Cfg(width=N, height=N, alpha_min=0.0)
    p = _prims2d((128.0, 128.0), (sig * sig, 0.0, sig * sig), f=f, c=(1, 1, 1))
    img = ora.forward(cfg, p)["color"][:, 0].reshape(N, N)
    F = np.abs(np.fft.fft2(img))
    ky = np.fft.fftfreq(N) * N
    kx = np.fft.fftfreq(N) * N
    KX, KY = np.meshgrid(kx, ky)
    rdc = 3 * N / (2 * math.pi * sig)
    Fm = np.where(np.hypot(KX, KY) > rdc, F, 0.0)
    iy, ix = np.unravel_index(np.argmax(Fm), F.shape)
    pk = np.array([kx[ix], ky[iy]])
    target = f * N / (2 * math.pi)
    assert min(np.linalg.norm(pk - target), np.linalg.norm(pk + target)) <= 1.0 + 1e-9
    # analytic spectrum (continuous FT, sampled at bin frequencies)
    wx, wy = 2 * math.pi * KX / N, 2 * math.pi * KY / N
    Sig = np.diag([sig * sig, sig * sig])

    def Ghat(ox, oy):
        return 2 * math.pi * math.sqrt(np.linalg.det(Sig)) * np.exp(
            -0.5 * (Sig[0, 0] * ox * ox + Sig[1, 1] * oy * oy))

    An = 0.5 * Ghat(wx, wy) + 0.25 * (Ghat(wx - f[0], wy - f[1]) + Ghat(wx + f[0], wy + f[1]))
    top = np.argsort(F.ravel())[-3:]
    np.testing.assert_allclose(F.ravel()[top], An.ravel()[top], rtol=0.02)


# ----------------------------------------------------------- tiling lemma
@pytest.mark.parametrize("tile", [8, 16, 32])
def test_tiled_equals_untiled_opacity_extent(ora, tile):
    """North-star 'tiled and untiled sums are equal' (lemma O3, R7):
    with the opacity-aware extent, adding the 'pixel's tile in rect' predicate
    changes nothing, bit for bit, in SUM and ALPHA modes."""
    H, W = 48, 64
    for blend in (False, True):
        p = gen.gen2d(H, W, 150, seed=11 + tile, freq_std=0.5, alpha=(0.3, 1.0), depth=True)
        pd = {k: v.astype(np.float64) for k, v in p.items()}
        cu = ora.Cfg(width=W, height=H, tile=tile, alpha_blend=blend)
        ct = ora.Cfg(width=W, height=H, tile=tile, alpha_blend=blend, use_rect=True)
        a = ora.forward(cu, pd)
        b = ora.forward(ct, pd)
        assert np.array_equal(a["color"], b["color"])
        assert np.array_equal(a["T"], b["T"])


def test_every_contributing_pair_is_binned(ora):
    """Lemma O3 by brute force: every (pixel, primitive) with alpha W >= alpha_min
    lies in a tile of the primitive's rect (SPEC S:237 'every primitive-tile pair
    with kernel support overlap appears ... in that tile's list')."""
    H, W = 64, 64
    p = gen.gen2d(H, W, 256, seed=1, freq_std=0.5)
    pd = {k: v.astype(np.float64) for k, v in p.items()}
    cfg = ora.Cfg(width=W, height=H)
    pr = ora.project2d(cfg, pd)
    ys, xs = np.mgrid[0:H, 0:W] + 0.5
    for i in range(256):
        if pr.flag[i]:
            continue
        r = pr.rec[i]
        dx, dy = xs - r[0], ys - r[1]
        q = r[2] * dx * dx + 2 * r[3] * dx * dy + r[4] * dy * dy
        w = r[12] * np.exp(-0.5 * q) * 0.5 * (1 + np.cos(r[5] * dx + r[6] * dy))
        yy, xx = np.nonzero(w >= cfg.alpha_min)
        tx, ty = xx // 16, yy // 16
        x0, y0, x1, y1 = pr.rect[i]
        assert np.all((tx >= x0) & (tx < x1) & (ty >= y0) & (ty < y1))


def test_bin_sort_integer_artifacts(ora):
    """O6: counts are rect areas; keys ascending; values within a tile in index
    order (SUM) or (depth, index) order (ALPHA); CSR offsets partition the list."""
    H, W = 64, 80
    for blend in (False, True):
        p = gen.gen2d(H, W, 300, seed=2, depth=True)
        pd = {k: v.astype(np.float64) for k, v in p.items()}
        cfg = ora.Cfg(width=W, height=H, alpha_blend=blend)
        pr = ora.project2d(cfg, pd)
        b = ora.bin_sort(cfg, pr)
        areas = np.maximum(pr.rect[:, 2] - pr.rect[:, 0], 0) * np.maximum(pr.rect[:, 3] - pr.rect[:, 1], 0)
        assert np.array_equal(pr.count, areas * (pr.flag == 0))
        assert b["total"] == areas[pr.flag == 0].sum()
        assert np.all(np.diff(b["keys"].astype(np.float64)) >= 0)
        GX, GY = -(-W // 16), -(-H // 16)
        toff = b["tile_offsets"]
        assert toff[0] == 0 and toff[-1] == b["total"] and np.all(np.diff(toff) >= 0)
        for u in range(GX * GY):
            seg = b["vals"][toff[u]:toff[u + 1]]
            assert np.all((b["keys"][toff[u]:toff[u + 1]] >> np.uint64(32)) == u)
            ty, tx = divmod(u, GX)
            expect = [i for i in range(300) if pr.flag[i] == 0 and pr.rect[i, 0] <= tx < pr.rect[i, 2]
                      and pr.rect[i, 1] <= ty < pr.rect[i, 3]]
            if blend:
                expect.sort(key=lambda i: (pr.keylo[i], i))
            assert list(seg) == expect


def test_sigma3_extent_is_tiling_dependent(ora):
    """DESIGN.md R7: SPEC's 3-sigma square makes the result depend on
    the tiling once alpha -> 1 (documented compatibility mode)."""
    H, W = 64, 64
    p = gen.gen2d(H, W, 300, seed=4, alpha=1.0, freq_std=0.0)
    pd = {k: v.astype(np.float64) for k, v in p.items()}
    a = ora.forward(ora.Cfg(width=W, height=H, tile=8, extent="sigma3"), pd)["color"]
    b = ora.forward(ora.Cfg(width=W, height=H, tile=32, extent="sigma3"), pd)["color"]
    c = ora.forward(ora.Cfg(width=W, height=H, tile=8), pd)["color"]
    d = ora.forward(ora.Cfg(width=W, height=H, tile=32), pd)["color"]
    assert not np.array_equal(a, b)
    assert np.array_equal(c, d)


RECTS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rect_examples.json")))


@pytest.mark.parametrize("ex", RECTS["cases"])
def test_tile_rect_hand_computed(ora, ex):
    """O1 steps 6-7 (R7; SPEC S:248 for the 3-sigma square): the
    oracle's tile rect equals a hand-computed one (tests/golden/rect_examples.json)
    placed so that an extent 5-10% too large or too small moves an edge —
    the tightness pin that the soundness lemma (every contributing pair is
    binned) cannot give."""
    p = dict(mean=np.array([ex["mean"]], np.float64), cov=np.array([ex["cov"]], np.float64),
             freq=np.zeros((1, 2)), color=np.ones((1, 3)) * 0.1,
             opacity=np.array([ex["alpha"]], np.float64))
    cfg = ora.Cfg(width=128, height=128, extent=ex["extent"])
    pr = ora.project2d(cfg, p)
    assert pr.flag[0] == 0
    assert list(pr.rect[0]) == ex["rect"], (list(pr.rect[0]), ex["derivation"])
    x0, y0, x1, y1 = ex["rect"]
    assert pr.count[0] == (x1 - x0) * (y1 - y0)


@pytest.mark.parametrize("blend", [False, True])
def test_render_counts(ora, blend):
    """The roofline work counters (ora_render_counts) against
    independent routes: SUM candidates = sum over tiles of list length x
    pixels of the tile (from the CSR offsets of bin_sort); contributing pairs =
    the forward's own per-pixel composited/contributing count (ncomp);
    cand >= ell >= con per pixel; without truncation of the list (T_min = 0)
    the ALPHA candidates are the whole tile lists."""
    H, W, N = 40, 56, 300
    p = gen.gen2d(H, W, N, seed=9, freq_std=0.2, alpha=(0.8, 1.0), color_max=1.0, depth=True,
                  s0=4.0)
    pd = {k: v.astype(np.float64) for k, v in p.items()}
    GX, GY = -(-W // 16), -(-H // 16)
    for tmin in (float(np.float32(1e-4)), 0.0):
        cfg = ora.Cfg(width=W, height=H, alpha_blend=blend, use_rect=True, T_min=tmin)
        pr = ora.project2d(cfg, pd)
        oc = ora.render_counts(cfg, pr, cfg.alpha_min * 2.0 ** -1e-4)
        ro = ora.render(cfg, pr)
        assert np.array_equal(oc["con"], ro["ncomp"].astype(np.int64))
        assert np.all(oc["cand"] >= oc["ell"]) and np.all(oc["ell"] >= oc["con"])
        toff = ora.bin_sort(cfg, pr)["tile_offsets"]
        ys, xs = np.divmod(np.arange(H * W), W)
        listlen = (toff[1:] - toff[:-1])[(ys // 16) * GX + xs // 16]
        if not blend or tmin == 0.0:
            assert np.array_equal(oc["cand"], listlen)
        else:
            assert np.all(oc["cand"] <= listlen) and np.any(oc["cand"] < listlen)

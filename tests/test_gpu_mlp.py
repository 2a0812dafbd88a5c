"""GPU parity of the NEXT-4 deformation field (tcgen05 MLP) against the FP64
oracle (oracle/mlp.py, pinned by torch autograd and FD in
tests/test_oracle_mlp.py).

precision="bf16x3" (the default, R38): against the UNQUANTIZED FP64
network (the FP32 D-3DGS lineage). A split-bf16 pair carries a
value to 2^-18 relative (|v - hi - lo| <= 2^-9 |v - hi| <= 2^-18 |v|), a product
drops lo.lo (<= 2^-18 relative): three roundings of 2^-18 per layer (operand,
weight, dropped term; fp32 accumulation is 2^-24), compounding over the D + 1
layers: u = 3 (D + 1) 2^-18 relative per output. Forward deltas: max error
<= 8 u of their rms (the max over up to 6e4 outputs of a per-output error of
rms u); gradients (dL/dz is re-split at every layer, a fourth rounding):
norm-wise tolG = 4 u, element-wise tolG |ref| + 8 tolG rms.

precision="bf16" (R36): both sides use the same bf16-rounded weights,
encoding and layer activations (the oracle's quantize=True rounds at the same
points, so the ReLU masks are decided on the same operands) and the oracle
accumulates in FP64. What remains on the GPU side is fp32 accumulation and, in
the backward, bf16 rounding of dL/dout and of each dL/dz (relative 2^-9 per
layer): forward deltas within 2e-2 of their rms, gradients within a norm-wise
2 (D + 1) 2^-9 (see _grad_ok).
"""
import numpy as np
import pytest

from oracle import mlp as omlp
from paper_2508_12615_b200 import gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_12615_b200 import build
    build.build()


def _bf16_round(x):
    t = torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).float()
    return t.numpy().astype(np.float64)


def _theta_as_kernel_sees_it(d, theta):
    """Weights rounded to bf16 (operands), biases kept fp32."""
    c = omlp.config(d.width, d.depth, d.skip, d.Lx, d.Lt)
    th = theta.cpu().numpy().astype(np.float64)
    out = th.copy()
    for name, shape, o in omlp.layout(c):
        if name.startswith("W"):
            n = int(np.prod(shape))
            out[o:o + n] = _bf16_round(th[o:o + n])
    return c, out


def _rel_ok(got, ref, frac=2e-2):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    rms = np.sqrt(np.mean(ref ** 2)) + 1e-30
    err = np.abs(got - ref)
    return float(np.max(err) / rms), bool(np.all(err <= frac * rms))


def _u3(depth):
    return 3 * (depth + 1) * 2.0 ** -18


def _grad_ok(got, ref, depth, tol=None):
    """Backward: dL/dz is rounded to bf16 at every layer on the GPU, a relative
    2^-9 per layer, so the gradient of layer l carries up to ~(D - l) 2^-9;
    bound (R36): norm-wise tol = 2 (D + 1) 2^-9, element-wise
    tol |ref| + 8 tol rms. The relative term matters at many rows: an entry fed
    by a constant-sign input column (t, the x coordinates) sums coherently over
    the rows and outgrows the rms by ~sqrt(rows), while its rounding error stays
    relative to itself."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    nrm = np.linalg.norm(ref) + 1e-30
    rel = float(np.linalg.norm(got - ref) / nrm)
    if tol is None:
        tol = 2 * (depth + 1) * 2.0 ** -9
    rms = nrm / np.sqrt(ref.size)
    return rel, rel <= tol and bool(np.all(np.abs(got - ref) <= tol * np.abs(ref) + 8 * tol * rms))


SHAPES = [dict(width=256, depth=8, skip=4, Lx=10, Lt=6),
          dict(width=64, depth=3, skip=0, Lx=4, Lt=2),
          dict(width=128, depth=2, skip=-1, Lx=10, Lt=6)]


@pytest.mark.parametrize("precision", ["bf16x3", "bf16"])
@pytest.mark.parametrize("shape", SHAPES)
def test_mlp_forward_backward_parity(shape, precision):
    _mlp_parity(shape, 1000, [0.0, 0.37, 1.0], precision)


@pytest.mark.parametrize("precision", ["bf16x3", "bf16"])
def test_mlp_parity_many_tiles_per_cta(precision):
    """40,000 rows (313 row tiles, ragged): every CTA pair of the fused layer
    backward accumulates dW over several tiles and cycles its operand rings."""
    _mlp_parity(dict(width=256, depth=8, skip=4, Lx=10, Lt=6), 20000, [0.25, 0.75], precision)


def _mlp_parity(shape, N, times, precision="bf16x3"):
    from paper_2508_12615_b200.deform import Deformation
    d = Deformation(N, **shape, precision=precision)
    theta = d.init_theta(seed=1)
    p = gen.gen3d(N, seed=3, scale_mult=4.0)
    canon = {k: torch.from_numpy(p[k]).cuda() for k in ("mean", "quat", "scale", "freq",
                                                         "color", "opacity")}
    frame = d.forward(theta, canon, times)
    torch.cuda.synchronize()
    x3 = precision == "bf16x3"
    if x3:  # the unquantized FP64 network
        c = omlp.config(d.width, d.depth, d.skip, d.Lx, d.Lt)
        th = theta.cpu().numpy().astype(np.float64)
    else:
        c, th = _theta_as_kernel_sees_it(d, theta)
    ref, cache = omlp.deform(c, th, {k: p[k] for k in ("mean", "quat", "scale", "freq")}, times,
                             quantize=not x3)
    frac = 8 * _u3(d.depth) if x3 else 2e-2
    gtol = 4 * _u3(d.depth) if x3 else None
    errs = {}
    for k in ("mean", "quat", "freq"):  # additive deltas: dx, dq, df
        delta_g = frame[k].cpu().numpy() - np.tile(p[k], (len(times), 1))
        delta_o = ref[k] - np.tile(p[k].astype(np.float64), (len(times), 1))
        worst, ok = _rel_ok(delta_g, delta_o, frac)
        errs[k] = worst
        assert ok, (k, worst, frac)
    # scale: compare the network output ds = log(s_t / s)
    ds_g = np.log(frame["scale"].cpu().numpy().astype(np.float64) / np.tile(p["scale"], (len(times), 1)))
    worst, ok = _rel_ok(ds_g, cache["out"][:, 7:10], frac)
    errs["scale"] = worst
    print(f"[mlp] {precision} {shape} N={N}: forward max err / rms {errs} (bound {frac:.2e})")
    assert ok, ("scale", worst)
    np.testing.assert_array_equal(frame["color"].cpu().numpy(), np.tile(p["color"], (len(times), 1)))
    # backward from a random upstream gradient of the frame rows
    rng = np.random.default_rng(5)
    gfr = {k: rng.normal(size=frame[k].shape).astype(np.float32)
           for k in ("mean", "quat", "scale", "freq")}
    if x3:
        # rows with a pre-activation within the forward's error (u of its layer's
        # rms) of the ReLU kink may take the other side of it on the GPU: both
        # derivatives are correct there (R25), so those rows get no upstream
        # gradient (the same protocol as the rasterizer's masked pixels, R24)
        P = omlp.unpack(c, th)
        amb = np.zeros(cache["ins"][0].shape[0], bool)
        for l in range(d.depth):
            z = cache["ins"][l] @ P[f"W{l}"].T + P[f"b{l}"]
            amb |= np.any(np.abs(z) < _u3(d.depth) * np.sqrt(np.mean(z * z)), axis=1)
        for k in gfr:
            gfr[k][amb] = 0.0
        print(f"[mlp] bf16x3: {int(amb.sum())} of {amb.size} rows near a ReLU kink excluded")
    g_theta, g_canon = d.backward(theta, canon, {k: torch.from_numpy(v).cuda()
                                                 for k, v in gfr.items()})
    torch.cuda.synchronize()
    gth_o, gcn_o = omlp.deform_backward(c, th, p, cache, gfr)
    gth = g_theta.cpu().numpy()
    bad, worst_all = [], 0.0
    for name, shp, o in omlp.layout(c):
        n = int(np.prod(shp))
        worst, ok = _grad_ok(gth[o:o + n], gth_o[o:o + n], d.depth, gtol)
        worst_all = max(worst_all, worst)
        if not ok:
            bad.append((name, round(worst, 6)))
    print(f"[mlp] {precision}: worst norm-wise gradient error {worst_all:.3e}")
    assert not bad, bad
    np.testing.assert_allclose(g_canon["mean"].cpu().numpy(), gcn_o["mean"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(g_canon["quat"].cpu().numpy(), gcn_o["quat"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(g_canon["freq"].cpu().numpy(), gcn_o["freq"], rtol=1e-5, atol=1e-5)
    worst, ok = _grad_ok(g_canon["scale"].cpu().numpy(), gcn_o["scale"], d.depth, gtol)
    assert ok, ("scale", worst)


def test_mlp_feeds_the_rasterizer():
    """6D end to end: deformation -> rasterizer (view_stride = N) -> backward
    through both, finite gradients everywhere (NEXT-4 'feeding K2 through
    view_stride')."""
    from paper_2508_12615_b200.deform import Deformation
    from paper_2508_12615_b200.raster import Rasterizer
    N, H, W = 2000, 96, 128
    p = gen.gen3d(N, seed=0, scale_mult=4.0)
    cams = gen.arc_cameras(3, W, H)
    canon = {k: torch.from_numpy(v).cuda() for k, v in p.items()}
    d = Deformation(N)
    theta = d.init_theta(seed=0, head_scale=0.1)
    frame = d.forward(theta, canon, [0.0, 0.5, 1.0])
    r = Rasterizer(W, H, prim="3d", blend="alpha")
    out = r.forward(frame, cams, view_stride=N)
    dL = torch.from_numpy(gen.gen_dLdC(3, H, W, seed=0)).cuda()
    gfr = r.backward(dL)
    g_theta, g_canon = d.backward(theta, canon, gfr)
    torch.cuda.synchronize()
    assert torch.isfinite(out["image"]).all()
    assert torch.isfinite(g_theta).all() and g_theta.abs().sum() > 0
    for v in g_canon.values():
        assert torch.isfinite(v).all()


@pytest.mark.parametrize("fused_train,N", [(False, 1000), (True, 1000), (True, 1), (True, 65)])
def test_mlp_inference_and_fused_paths_agree(fused_train, N, tmp_path):
    """The fused on-chip forward (mlp_fused.cu; used for train=False, and for
    training with WIPES_MLP_FUSED=1) gives the same frame rows as the
    layer-by-layer schedule up to fp32 accumulation order; with training on,
    its stored activations drive the same backward. WIPES_MLP_UNFUSED=1 also
    turns off the fused layer kernels (k_mlp_fwd_layer, k_mlp_bwd_layer), so
    2 and 130 rows cover their single-tile and ragged edge cases."""
    import os
    import subprocess
    import sys
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {os.getcwd()!r})
from paper_2508_12615_b200 import gen
from paper_2508_12615_b200.deform import Deformation
N = {N}
d = Deformation(N, precision="bf16")
th = d.init_theta(2)
p = gen.gen3d(N, seed=4)
canon = {{k: torch.from_numpy(v).cuda() for k, v in p.items()}}
f = d.forward(th, canon, [0.1, 0.9], train={fused_train})
g = {{k: torch.ones_like(f[k]) for k in ("mean", "quat", "scale", "freq")}}
out = {{k: v.cpu().numpy() for k, v in f.items()}}
if {fused_train}:
    gt, gc = d.backward(th, canon, g)
    out["g_theta"] = gt.cpu().numpy()
np.savez(sys.argv[1], **out)
"""
    res = {}
    for tag, env in (("fused", {"WIPES_MLP_FUSED": "1"}), ("unfused", {"WIPES_MLP_UNFUSED": "1"})):
        path = str(tmp_path / f"mlp_{tag}.npz")
        e = {k: v for k, v in os.environ.items() if not k.startswith("WIPES_MLP_")}
        e.update(env)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=e, timeout=300)
        res[tag] = np.load(path)
    for k in ("mean", "quat", "scale", "freq", "color", "opacity"):
        a, b = res["fused"][k].astype(np.float64), res["unfused"][k].astype(np.float64)
        np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-5 * (np.abs(b).max() + 1e-30))
    if fused_train:
        a, b = res["fused"]["g_theta"], res["unfused"]["g_theta"]
        assert np.linalg.norm(a - b) <= 1e-3 * np.linalg.norm(b)


def test_autograd_deform_and_rasterize():
    """deform() and rasterize() compose under torch.autograd: one loss.backward()
    reaches theta and the canonical parameters through both libraries' kernels,
    and matches the explicit backward calls."""
    from paper_2508_12615_b200.deform import Deformation, deform
    from paper_2508_12615_b200.raster import Rasterizer, rasterize
    N, H, W = 1500, 64, 96
    p = gen.gen3d(N, seed=1, scale_mult=4.0)
    cams = gen.arc_cameras(2, W, H)
    d = Deformation(N)
    theta = d.init_theta(3, head_scale=0.1).requires_grad_(True)
    canon = {k: torch.from_numpy(v).cuda().requires_grad_(True) for k, v in p.items()}
    r = Rasterizer(W, H, prim="3d", blend="alpha")
    frame = deform(d, theta, canon, [0.2, 0.8])
    img = rasterize(r, frame, cams, view_stride=N)
    w = torch.from_numpy(gen.gen_dLdC(2, H, W, seed=5)).cuda()
    (img * w).sum().backward()
    assert theta.grad is not None and torch.isfinite(theta.grad).all()
    # explicit path
    fr = d.forward(theta.detach(), {k: v.detach() for k, v in canon.items()}, [0.2, 0.8])
    r2 = Rasterizer(W, H, prim="3d", blend="alpha")
    r2.forward(fr, cams, N)
    gfr = r2.backward(w)
    gt, gc = d.backward(theta.detach(), {k: v.detach() for k, v in canon.items()}, gfr)
    torch.cuda.synchronize()
    assert torch.linalg.norm(theta.grad - gt) <= 1e-4 * torch.linalg.norm(gt) + 1e-12
    for k in ("mean", "quat", "scale", "freq"):
        assert torch.linalg.norm(canon[k].grad - gc[k]) <= 1e-4 * torch.linalg.norm(gc[k]) + 1e-12
    assert torch.linalg.norm(canon["color"].grad - gfr["color"].reshape(2, N, 3).sum(0)) <= \
        1e-5 * torch.linalg.norm(gfr["color"]) + 1e-12


def test_mlp_forward_bitwise_deterministic():
    """The forward (layer kernels, TMA stores, no atomics) is bitwise
    reproducible run to run; the backward agrees to rounding level (the
    weight-gradient GEMMs of the head, layer 0 and the encoding columns after
    the skip accumulate split-K partials with fp32 atomics)."""
    from paper_2508_12615_b200.deform import Deformation
    N = 9000
    d = Deformation(N)
    th = d.init_theta(4)
    p = gen.gen3d(N, seed=6)
    canon = {k: torch.from_numpy(v).cuda() for k, v in p.items()}
    outs = []
    for _ in range(2):
        f = d.forward(th, canon, [0.3, 0.6])
        g = {k: torch.ones_like(f[k]) for k in ("mean", "quat", "scale", "freq")}
        gt, gc = d.backward(th, canon, g)
        torch.cuda.synchronize()
        outs.append(({k: v.clone() for k, v in f.items()}, gt.clone(), {k: v.clone() for k, v in gc.items()}))
    (f0, gt0, gc0), (f1, gt1, gc1) = outs
    for k in f0:
        assert torch.equal(f0[k], f1[k]), k
    assert torch.linalg.norm(gt0 - gt1) <= 1e-5 * torch.linalg.norm(gt0)
    for k in gc0:
        assert torch.linalg.norm(gc0[k] - gc1[k]) <= 1e-5 * torch.linalg.norm(gc0[k]) + 1e-12, k


def test_deformed_6d_image_against_fp64_network(ora):
    """NEXT-4 faithful end to end (R38): the split-bf16 deformation
    field feeding the rasterizer (view_stride = N) against the UNQUANTIZED FP64
    network feeding the FP64 oracle rasterizer. The network's error is carried
    to the image by re-rendering the GPU's own frame rows in the oracle:
    |I_gpu - I_fp64| <= pixel tolerance (rasterizer parity, R23) +
    |I_oracle(GPU rows) - I_oracle(FP64 rows)| (the propagated network error),
    and that propagated error must stay below the pixel tolerance itself."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from parity_util import oracle_cfg, pixel_violations
    from paper_2508_12615_b200.deform import Deformation
    from paper_2508_12615_b200.raster import Rasterizer
    N, H, W, times = 2000, 96, 128, [0.0, 0.5, 1.0]
    B = len(times)
    p = gen.gen3d(N, seed=0, scale_mult=4.0)
    cams = gen.arc_cameras(B, W, H)
    d = Deformation(N)
    assert d.precision == "bf16x3"
    theta = d.init_theta(seed=0, head_scale=0.1)
    canon = {k: torch.from_numpy(v).cuda() for k, v in p.items()}
    frame = d.forward(theta, canon, times)
    r = Rasterizer(W, H, prim="3d", blend="alpha")
    img = r.forward(frame, cams, view_stride=N)["image"]
    torch.cuda.synchronize()
    c = omlp.config(d.width, d.depth, d.skip, d.Lx, d.Lt)
    th = theta.cpu().numpy().astype(np.float64)
    ref, _ = omlp.deform(c, th, {k: p[k] for k in ("mean", "quat", "scale", "freq")}, times,
                         quantize=False)
    rows_o = {k: np.ascontiguousarray(ref[k].astype(np.float32)) for k in ref}
    rows_g = {k: frame[k].cpu().numpy() for k in ("mean", "quat", "scale", "freq")}
    for k in ("color", "opacity"):
        rows_o[k] = rows_g[k] = frame[k].cpu().numpy()
    cfg_o = oracle_cfg(ora, "3d", H, W, "alpha", use_rect=True)
    pr_o = ora.project3d(cfg_o, rows_o, cams, view_stride=N)
    pr_g = ora.project3d(cfg_o, rows_g, cams, view_stride=N)
    ro_o, ro_g = ora.render(cfg_o, pr_o), ora.render(cfg_o, pr_g)
    got = img.cpu().numpy().transpose(0, 2, 3, 1).reshape(-1, 3)
    prop = np.abs(ro_o["color"] - ro_g["color"])
    amb = np.minimum(ro_o["margin"], ro_g["margin"])
    nb, namb = pixel_violations(got, ro_g["color"], amb)
    assert nb == 0, (nb, namb)
    keep = amb >= 1e-5
    err = np.abs(got - ro_o["color"])
    tol = np.maximum(1e-5, 1e-4 * np.abs(ro_o["color"])) + prop
    print(f"[mlp] 6D image: max |I_gpu - I_fp64| {err[keep].max():.3e}, propagated network "
          f"error max {prop[keep].max():.3e}, masked px {int((~keep).sum())}")
    assert np.all(err[keep] <= tol[keep])
    assert np.all(prop[keep] <= np.maximum(1e-5, 1e-4 * np.abs(ro_o["color"][keep])))

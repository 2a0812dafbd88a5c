"""GPU parity: the CUDA path (through the C ABI) against the double-precision
oracle on the same seeded float32 inputs (run with `pytest -m gpu` on a B200).

Integer artefacts (tile rects, counts, offsets, sorted keys/values, per-tile
CSR ranges, cull flags) must be bit-exact. Pixels: |g - o| <= max(1e-5,
1e-4 |o|); gradients: |g - o| <= max(1e-5, 1e-3 |o|) (north_star; DESIGN.md
R23), with threshold-ambiguous pixels (decision margin < 1e-5) masked and
counted (R24). Gradients follow SURVEY §8(c)'s protocol: the rows
(primitives, or (view, primitive) for per-frame sets) with a pair at a masked
pixel are excluded and counted, every other row must meet the tolerance with
zero violations (tests/parity_util.py check_grads_strict prints both counts).
"""
import numpy as np
import pytest

from paper_2508_12615_b200 import gen
from parity_util import (oracle_cfg, gpu_rasterizer, to_dev, pixel_violations,
                         grad_violations, f32, ambiguous_rows, check_grads_strict,
                         oracle_grads)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_12615_b200 import build
    build.build()


def _np(t):
    return t.detach().cpu().numpy()


def _check_integers(ora, cfg_o, pr, r, B, N):
    pre = r.get_preprocess()
    torch.cuda.synchronize()
    assert np.array_equal(_np(pre["rect"]), pr.rect.reshape(B * N, 4)), "tile rects differ"
    assert np.array_equal(_np(pre["count"]), pr.count), "tile counts differ"
    b = ora.bin_sort(cfg_o, pr)
    assert np.array_equal(_np(pre["offsets"]), b["offsets"]), "offsets differ"
    if cfg_o.alpha_blend:
        dk = _np(pre["depth_key"]).view(np.uint32)
        live = pr.flag == 0
        assert np.array_equal(dk[live], pr.keylo[live]), "depth keys differ"
    keys, vals, toff = r.bin_sort_outputs()
    torch.cuda.synchronize()
    assert keys.shape[0] == b["total"]
    assert np.array_equal(_np(keys).view(np.uint64), b["keys"]), "sorted keys differ"
    assert np.array_equal(_np(vals).view(np.uint32), b["vals"]), "sorted values differ"
    assert np.array_equal(_np(toff).astype(np.int64), b["tile_offsets"]), "tile ranges differ"
    return b


def _pixels(arr_bchw):
    a = np.asarray(arr_bchw)
    return a.transpose(0, 2, 3, 1).reshape(-1, 3)


# --------------------------------------------------------------------- 2D --
@pytest.mark.parametrize("cov2", ["sigma", "cholesky", "rs"])
@pytest.mark.parametrize("blend", ["sum", "alpha"])
def test_c1_2d_full_parity(ora, cov2, blend):
    """configs[0] (C1): 64x64, 256 primitives — every integer artefact
    bit-exact, every pixel and every gradient within tolerance."""
    H = W = 64
    N = 256
    p = gen.gen2d(H, W, N, seed=0, cov_mode=cov2, freq_std=0.5, phase=True,
                  alpha=(0.2, 1.0) if blend == "alpha" else 1.0,
                  color_max=1.0 if blend == "alpha" else 0.1, depth=(blend == "alpha"))
    cfg_o = oracle_cfg(ora, "2d", H, W, blend, cov2=cov2)
    pr = ora.project2d(cfg_o, p)
    r = gpu_rasterizer("2d", H, W, blend, cov2=cov2)
    dp = to_dev(p)
    out = r.forward(dp)
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, 1, N)
    dL = gen.gen_dLdC(1, H, W, seed=0)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    img = _pixels(_np(out["image"]))
    nbad, namb = pixel_violations(img, ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    assert namb <= 4
    if blend == "alpha":
        nbad, _ = pixel_violations(_np(out["T_final"]).reshape(-1), ro["T"], ro["margin"])
        assert nbad == 0
    grads = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro)
    exc = ambiguous_rows(pr, ro["margin"], 1, N, H, W)
    check_grads_strict(grads, og, exc, f"C1 {cov2} {blend}",
                       keys=("mean", "cov", "freq", "phase", "color", "opacity"), bound=gb)


@pytest.mark.parametrize("tile", [8, 32])
def test_tile_size_invariance_bitwise(tile):
    """Lemma O3 on the GPU: images rendered with 8/16/32-pixel tiles are bit
    for bit identical (same per-pixel contributor set and order, R7)."""
    H, W = 96, 80
    for blend in ("sum", "alpha"):
        p = gen.gen2d(H, W, 500, seed=3, freq_std=0.5, phase=True, alpha=(0.2, 1.0),
                      depth=(blend == "alpha"))
        dp = to_dev(p)
        a = gpu_rasterizer("2d", H, W, blend, tile=16).forward(dp)["image"]
        b = gpu_rasterizer("2d", H, W, blend, tile=tile).forward(dp)["image"]
        torch.cuda.synchronize()
        assert torch.equal(a, b), (blend, tile)


def test_c2_kodak_integer_and_sampled_parity(ora):
    """configs[1] (C2, the bench workload): 768x512, 70k primitives. Integer
    artefacts bit-exact; pixels and gradients on 4096 sampled pixels (dL/dC is
    non-zero only there, so the oracle's subset gradient is the full one)."""
    c = gen.make_config("c2", seed=0)
    H, W, N = c["H"], c["W"], c["N"]
    p = c["params"]
    cfg_o = oracle_cfg(ora, "2d", H, W, "sum", use_rect=True)
    pr = ora.project2d(cfg_o, p)
    r = gpu_rasterizer("2d", H, W, "sum")
    out = r.forward(to_dev(p))
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, 1, N)
    rng = np.random.default_rng(7)
    pix = np.sort(rng.choice(H * W, 4096, replace=False))
    dLfull = np.zeros((1, 3, H, W), np.float32)
    dLs = rng.uniform(-1, 1, (4096, 3)).astype(np.float32)
    dLfull[0, :, pix // W, pix % W] = dLs
    ro = ora.render(cfg_o, pr, pix=pix, dLdC=dLs, abs_terms=True)
    img = _pixels(_np(out["image"]))[pix]
    nbad, namb = pixel_violations(img, ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    grads = r.backward(torch.from_numpy(dLfull).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro)
    exc = ambiguous_rows(pr, ro["margin"], 1, N, H, W, pix=pix)
    check_grads_strict(grads, og, exc, "C2 sampled",
                       keys=("mean", "cov", "freq", "color", "opacity"), bound=gb)


# --------------------------------------------------------------------- 3D --
@pytest.mark.parametrize("name", ["p3d", "p6d"])
def test_mini_3d_6d_parity(ora, name):
    """Parity-only mini configs: 3D static (2 views, shared
    params) and 6D per-frame params (view_stride = N)."""
    c = gen.make_config(name, seed=0)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    cfg_o = oracle_cfg(ora, "3d", H, W, "alpha", use_rect=True)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    r = gpu_rasterizer("3d", H, W, "alpha")
    cull = torch.zeros(B * N, dtype=torch.uint8, device="cuda")
    r.preprocess(to_dev(p), cams, view_stride=vs, cull_flags=cull)
    r.bin_sort()
    img, T, nc = r.render()
    torch.cuda.synchronize()
    assert np.array_equal(_np(cull), pr.flag.astype(np.uint8)), "cull flags differ"
    _check_integers(ora, cfg_o, pr, r, B, N)
    dL = gen.gen_dLdC(B, H, W, seed=1)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    nbad, namb = pixel_violations(_pixels(_np(img)), ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    assert namb <= 0.002 * B * H * W
    grads = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    check_grads_strict(grads, og, exc, f"{name} alpha",
                       keys=("mean", "scale", "quat", "freq", "color", "opacity"), bound=gb)


@pytest.mark.parametrize("blend", ["alpha", "sum"])
def test_f64_moment_accumulation_parity(ora, blend):
    """cfg.grad_accum = WIPES_ACCUM_F64 (R37): FP64 lane sums, exact
    products and FP64 warp reduction of the backward moments. Same protocol as
    the FP32 default. The aggregate errors of both are printed: they are equal
    to within a few percent (measured f32 0.141 / f64 0.142 at p3d ALPHA), i.e.
    the per-pair FP32/SFU evaluation, not the summation, sets the error (R23b)."""
    c = gen.make_config("p3d", seed=0)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    dL = gen.gen_dLdC(B, H, W, seed=3)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    errs = {}
    for acc in ("f32", "f64"):
        r = gpu_rasterizer("3d", H, W, blend, grad_accum=acc)
        r.forward(to_dev(p), cams, vs)
        grads = r.backward(torch.from_numpy(dL).cuda())
        torch.cuda.synchronize()
        check_grads_strict(grads, og, exc, f"p3d {blend} grad_accum={acc}", bound=gb)
        errs[acc] = sum(float(np.sum(np.abs(_np(grads[k]) - og[k])[~exc]))
                        for k in ("mean", "scale", "quat"))
    print(f"[parity] p3d {blend}: sum |g - o| over mean/scale/quat: f32 {errs['f32']:.3e}, "
          f"f64 {errs['f64']:.3e}")
    assert errs["f64"] <= 1.25 * errs["f32"] and errs["f32"] <= 1.25 * errs["f64"]


@pytest.mark.parametrize("name,blend", [("p3d", "alpha"), ("p3d", "sum"), ("p6d", "alpha")])
def test_exact_projection_parity(ora, name, blend):
    """NEXT-1 exact z-integration (R4): f' and
    beta = exp(-1/2 f_hat_z^2 v) from the full ray-space covariance in the
    forward, the beta moment and the dual-number Jacobian of the exact
    projection in the backward, against the oracle's exact mode (whose chain is
    pinned by whole-pipeline finite differences, test_oracle_grad.py)."""
    c = gen.make_config(name, seed=0)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True, exact_proj=True)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    beta = pr.field("beta")[pr.flag == 0]
    assert np.median(beta) < 0.95  # the exact mode is exercised
    r = gpu_rasterizer("3d", H, W, blend, proj="exact")
    r.preprocess(to_dev(p), cams, view_stride=vs)
    r.bin_sort()
    img, T, nc = r.render()
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, B, N)
    dL = gen.gen_dLdC(B, H, W, seed=2)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    nbad, namb = pixel_violations(_pixels(_np(img)), ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    assert namb <= 0.002 * B * H * W
    grads = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    check_grads_strict(grads, og, exc, f"{name} {blend} exact",
                       keys=("mean", "scale", "quat", "freq", "color", "opacity"), bound=gb)


@pytest.mark.parametrize("name,blend,deg", [("p3d", "alpha", 3), ("p3d", "sum", 2),
                                             ("p6d", "alpha", 3), ("p3d", "alpha", 0)])
def test_sh_colour_parity(ora, name, blend, deg):
    """NEXT-3 SH colour: per-(view, primitive) colour from
    degree-`deg` SH in the FP64 preprocess; dL/dsh and the view-direction term
    of dL/dmu in k_sh_bwd, against the oracle (pinned by orthonormality and
    whole-pipeline FD, tests/test_oracle_sh.py)."""
    c = gen.make_config(name, seed=0, sh_degree=deg)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    assert "sh" in p and "color" not in p
    cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True, sh_degree=deg)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    r = gpu_rasterizer("3d", H, W, blend, sh_degree=deg)
    r.preprocess(to_dev(p), cams, view_stride=vs)
    r.bin_sort()
    img, T, nc = r.render()
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, B, N)
    rec = _np(r.get_preprocess()["records"]).reshape(B * N, 16)
    live = pr.flag == 0
    col_o = np.stack([pr.field("cr"), pr.field("cg"), pr.field("cb")], 1)
    np.testing.assert_allclose(rec[live, 12:15], col_o[live], rtol=1e-6, atol=1e-7)
    dL = gen.gen_dLdC(B, H, W, seed=4)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    nbad, namb = pixel_violations(_pixels(_np(img)), ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    grads = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    assert "color" not in og and og["sh"].shape == p["sh"].shape
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    check_grads_strict(grads, og, exc, f"{name} {blend} SH{deg}",
                       keys=("mean", "scale", "quat", "freq", "opacity", "sh"), bound=gb)


@pytest.mark.parametrize("kind,blend,extra", [("2d", "sum", {}), ("2d", "alpha", {}),
                                              ("3d", "alpha", {}), ("3d", "alpha",
                                                                    {"proj": "exact"})])
def test_deterministic_backward_bitwise_and_parity(ora, kind, blend, extra):
    """cfg.deterministic: two backward passes are bitwise equal and
    match the oracle like the atomic path; integer artefacts unchanged."""
    if kind == "2d":
        H = W = 64
        p = gen.gen2d(H, W, 256, seed=4, freq_std=0.5, phase=True, alpha=(0.2, 1.0),
                      color_max=1.0 if blend == "alpha" else 0.1, depth=(blend == "alpha"))
        cams, vs, B, N = None, 0, 1, 256
        cfg_o = oracle_cfg(ora, "2d", H, W, blend, use_rect=True)
    else:
        c = gen.make_config("p3d", seed=1)
        H, W, N, B = c["H"], c["W"], c["N"], c["B"]
        p, cams, vs = c["params"], c["cams"], c["view_stride"]
        cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True,
                           exact_proj=extra.get("proj") == "exact")
    r = gpu_rasterizer(kind, H, W, blend, deterministic=1, **extra)
    dp = to_dev(p)
    dL = gen.gen_dLdC(B, H, W, seed=7)
    outs = []
    for _ in range(2):
        out = r.forward(dp, cams, vs) if kind == "3d" else r.forward(dp)
        g = r.backward(torch.from_numpy(dL).cuda())
        torch.cuda.synchronize()
        outs.append((out["image"].clone(), {k: v.clone() for k, v in g.items()}))
    assert torch.equal(outs[0][0], outs[1][0])
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs) if kind == "3d" else ora.project2d(cfg_o, p)
    _check_integers(ora, cfg_o, pr, r, B, N)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    nbad_pix, namb = pixel_violations(_pixels(_np(outs[0][0])), ro["color"], ro["margin"])
    assert nbad_pix == 0
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    check_grads_strict(outs[0][1], og, exc, f"deterministic {kind} {blend} {extra}", bound=gb)


_EXACT_GRADS = """
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
from paper_2508_12615_b200 import gen
from parity_util import gpu_rasterizer, to_dev
c = gen.make_config('p3d', seed=0)
r = gpu_rasterizer('3d', c['H'], c['W'], 'alpha', proj='exact', deterministic=1)
r.forward(to_dev(c['params']), c['cams'])
g = r.backward(torch.from_numpy(gen.gen_dLdC(c['B'], c['H'], c['W'], seed=2)).cuda())
np.savez(sys.argv[2], **{k: v.cpu().numpy() for k, v in g.items()})
"""


def test_exact_adjoint_matches_forward_mode(tmp_path):
    """The hand-written adjoint of the exact projection (k_pre3d_bwd<EXACT>)
    against forward-mode dual-number differentiation of the same exact
    projection code (k_pre3d_bwd_exact, selected by WIPES_EXACT_DUAL)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag in ("adj", "dual"):
        f = str(tmp_path / f"{tag}.npz")
        e = {k: v for k, v in os.environ.items() if k != "WIPES_EXACT_DUAL"}
        if tag == "dual":
            e["WIPES_EXACT_DUAL"] = "1"
        subprocess.run([sys.executable, "-c", _EXACT_GRADS, root, f], check=True, env=e,
                       timeout=600)
        out[tag] = np.load(f)
    for k in out["adj"].files:
        a, d = out["adj"][k].astype(np.float64), out["dual"][k].astype(np.float64)
        # deterministic backward: the render moments are bitwise reproducible, so
        # the two runs differ only in the FP64 projection adjoint vs dual numbers
        # (with atomics their order alone moved cancelling sums past 1e-4)
        tol = 1e-5 + 1e-4 * np.abs(d)
        assert np.all(np.abs(a - d) <= tol), (k, np.max(np.abs(a - d) - tol))


# --------------------------------------------------------------- contract --
def test_capacity_protocol_overflow_then_retry():
    H = W = 64
    p = to_dev(gen.gen2d(H, W, 256, seed=1))
    r = gpu_rasterizer("2d", H, W, "sum")
    ref = r.forward(p)["image"].clone()
    total = r.n_dup
    r2 = gpu_rasterizer("2d", H, W, "sum")
    r2._alloc(256, 1, total // 2)
    r2.preprocess(p, sync=False)
    r2.bin_sort()
    r2.render()
    n, over = r2.check_overflow()
    assert n == total and over
    r2._alloc(256, 1, total)
    img = r2.forward(p, sync=False)["image"]
    n, over = r2.check_overflow()
    assert not over
    assert torch.equal(img, ref)


def test_empty_scene_and_all_culled():
    H = W = 32
    for blend, bg in (("sum", (0, 0, 0)), ("alpha", (0.1, 0.2, 0.3))):
        p = to_dev(gen.gen2d(H, W, 4, seed=2, depth=True))
        empty = {k: v[:0].contiguous() for k, v in p.items()}
        r = gpu_rasterizer("2d", H, W, blend, background=bg)
        out = r.forward(empty)
        torch.cuda.synchronize()
        for ch in range(3):
            assert torch.all(out["image"][0, ch] == f32(bg[ch]))
        # non-finite inputs are culled (flag 5), not errors
        bad = {k: v.clone() for k, v in p.items()}
        bad["mean"][:] = float("nan")
        cull = torch.zeros(4, dtype=torch.uint8, device="cuda")
        r2 = gpu_rasterizer("2d", H, W, blend, background=bg)
        r2.preprocess(bad, cull_flags=cull)
        torch.cuda.synchronize()
        assert torch.all(cull == 5)


def test_forward_run_to_run_deterministic():
    """The forward has no atomics (each pixel accumulates its list in order):
    repeated runs are bit-identical whatever the work scheduling."""
    H, W = 96, 80
    for blend in ("sum", "alpha"):
        dp = to_dev(gen.gen2d(H, W, 500, seed=4, freq_std=0.5, phase=True, depth=True))
        r = gpu_rasterizer("2d", H, W, blend)
        a = r.forward(dp)["image"].clone()
        for _ in range(3):
            b = r.forward(dp)["image"]
            torch.cuda.synchronize()
            assert torch.equal(a, b)


# ------------------------------------------------------- full-size configs --
@pytest.mark.parametrize("name", ["c3", "c5"])
def test_full_size_sampled_parity(ora, name):
    """BASELINE.json configs at full size (C3: 8 x 1080p views, 1M primitives,
    alpha blending; C5: 4K image, 3M primitives, weighted sum), in the bench's
    launch configuration: every integer artefact bit-exact against the oracle,
    pixels on 2048 sampled pixels (the oracle evaluates them one by one)."""
    c = gen.make_config(name, seed=0)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    kind = "2d" if c["kind"] == "2d" else "3d"
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    cfg_o = oracle_cfg(ora, kind, H, W, c["blend"], use_rect=True)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs) if kind == "3d" else ora.project2d(cfg_o, p)
    r = gpu_rasterizer(kind, H, W, c["blend"])
    out = r.forward(to_dev(p), cams, vs)
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, B, N)
    rng = np.random.default_rng(11)
    pix = np.sort(rng.choice(B * H * W, 2048, replace=False))
    ro = ora.render(cfg_o, pr, pix=pix)
    img = _pixels(_np(out["image"]))[pix]
    nbad, namb = pixel_violations(img, ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    if c["blend"] == "alpha":
        nbad, _ = pixel_violations(_np(out["T_final"]).reshape(-1)[pix], ro["T"], ro["margin"])
        assert nbad == 0


# ------------------------------------------------------ image-space sharding --
@pytest.mark.parametrize("blend", ["sum", "alpha"])
@pytest.mark.parametrize("world", [2, 3])
def test_row_sharding_equals_full(ora, blend, world):
    """SURVEY §8(e) tile-row sharding of one image: rank r bins and renders the
    tile rows ty = r (mod world). Its rows are bit-identical to the unsharded
    render (same per-tile lists, same order), its counts are the oracle's rects
    restricted to its rows, and the ranks' gradients sum to the full gradient."""
    H, W, N = 160, 144, 3000
    p = gen.gen2d(H, W, N, seed=5, freq_std=0.4, phase=True, alpha=(0.3, 1.0),
                  depth=(blend == "alpha"))
    dp = to_dev(p)
    dL = torch.from_numpy(gen.gen_dLdC(1, H, W, seed=5)).cuda()
    full = gpu_rasterizer("2d", H, W, blend)
    img = full.forward(dp)["image"].clone()
    gfull = {k: v.clone() for k, v in full.backward(dL).items()}
    cfg_o = oracle_cfg(ora, "2d", H, W, blend)
    pr = ora.project2d(cfg_o, p)
    gsum = None
    rows = (np.arange(H) // 16)
    for r in range(world):
        rs = gpu_rasterizer("2d", H, W, blend, row_mod=world, row_rem=r)
        out = rs.forward(dp)
        torch.cuda.synchronize()
        mask = torch.from_numpy(rows % world == r).cuda()
        assert torch.equal(out["image"][..., mask, :], img[..., mask, :])
        cnt = _np(rs.get_preprocess()["count"])
        nx = np.maximum(pr.rect[:, 2] - pr.rect[:, 0], 0)
        ny = np.array([sum(1 for ty in range(y0, y1) if ty % world == r)
                       for (_, y0, _, y1) in pr.rect])
        assert np.array_equal(cnt, nx * ny * (pr.flag == 0))
        g = rs.backward(dL)
        torch.cuda.synchronize()
        gsum = {k: v.clone() for k, v in g.items()} if gsum is None else \
            {k: gsum[k] + g[k] for k in g}
    for k in gfull:
        a, b = _np(gsum[k]), _np(gfull[k])
        assert np.allclose(a, b, rtol=1e-4, atol=1e-6), (k, np.abs(a - b).max())


@pytest.mark.parametrize("vs_mode,sh", [("shared", None), ("per_frame", None), ("shared", 2)])
def test_more_than_128_views(ora, vs_mode, sh):
    """B = 131 > WIPES_MAX_CAMERAS_PER_LAUNCH: the camera blocks are processed in
    chunks (preprocess, preprocess backward with accumulation across chunks,
    SH backward); results equal the oracle's."""
    N, B, H, W = 60, 131, 32, 32
    rng = np.random.default_rng(0)
    base = gen.gen3d(N, seed=2, scale_mult=20.0, sh_degree=sh)
    cams = [gen.camera((2.5 * np.cos(a), -0.3, 2.5 * np.sin(a)), W, H)
            for a in np.linspace(0, 2 * np.pi, B, endpoint=False)]
    if vs_mode == "per_frame":
        p = {k: np.concatenate([v] * B, 0) for k, v in base.items()}
        p["mean"] = (p["mean"] + rng.normal(0, 0.01, p["mean"].shape)).astype(np.float32)
        vs = N
    else:
        p, vs = base, 0
    cfg_o = oracle_cfg(ora, "3d", H, W, "alpha", use_rect=True, sh_degree=sh)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    r = gpu_rasterizer("3d", H, W, "alpha", sh_degree=sh)
    out = r.forward(to_dev(p), cams, vs)
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, B, N)
    dL = gen.gen_dLdC(B, H, W, seed=3)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    nbad, namb = pixel_violations(_pixels(_np(out["image"])), ro["color"], ro["margin"])
    assert nbad == 0
    grads = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    check_grads_strict(grads, og, exc, f"131 views {vs_mode} SH{sh}", bound=gb)


# --------------------------------------------------- partial tiles, counters --
@pytest.mark.parametrize("kind,blend", [("2d", "sum"), ("2d", "alpha"), ("3d", "alpha"),
                                        ("3d", "sum")])
def test_partial_tile_backward_parity(ora, kind, blend):
    """W and H not multiples of 16: the last tile column and
    row are partial, so the in-image guards of the forward AND backward
    (pixels outside the image neither written nor contributing) are compared
    with the oracle on every pixel and every gradient."""
    if kind == "2d":
        H, W, N, B = 70, 100, 400, 1
        p = gen.gen2d(H, W, N, seed=6, freq_std=0.5, phase=True, alpha=(0.2, 1.0),
                      color_max=1.0 if blend == "alpha" else 0.1, depth=(blend == "alpha"))
        cams, vs = None, 0
        cfg_o = oracle_cfg(ora, "2d", H, W, blend, use_rect=True)
        pr = ora.project2d(cfg_o, p)
    else:
        H, W, N, B = 90, 122, 4000, 2
        p = gen.gen3d(N, seed=3, scale_mult=6.0)
        cams = gen.ring_cameras(B, W, H)
        vs = 0
        cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True)
        pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
    r = gpu_rasterizer(kind, H, W, blend)
    out = r.forward(to_dev(p), cams, vs)
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, B, N)
    dL = gen.gen_dLdC(B, H, W, seed=8)
    ro = ora.render(cfg_o, pr, dLdC=_pixels(dL), abs_terms=True)
    nbad, namb = pixel_violations(_pixels(_np(out["image"])), ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    if blend == "alpha":
        nbad, _ = pixel_violations(_np(out["T_final"]).reshape(-1), ro["T"], ro["margin"])
        assert nbad == 0
    grads = r.backward(torch.from_numpy(dL).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs)
    check_grads_strict(grads, og, exc, f"partial tiles {kind} {blend} {W}x{H}", bound=gb)


@pytest.mark.parametrize("case", ["c1_sum", "c1_alpha", "p3d_alpha", "p3d_sum", "p6d_alpha"])
def test_render_stats_counters_match_oracle(ora, case):
    """The roofline's work units: wipes_render_stats' tile-method
    candidate pairs, in-ellipse pairs and contributing pairs against the
    oracle's per-pixel counts over each pixel's tile list
    (ora_render_counts). Candidates are integer bookkeeping and must be exact
    (up to the list tails of threshold-ambiguous pixels in ALPHA mode);
    in-ellipse and contributing counts may differ only by the pairs whose
    FP32 decision is within rounding of its threshold."""
    name, blend = case.split("_")
    if name == "c1":
        H = W = 64
        N, B = 256, 1
        p = gen.gen2d(H, W, N, seed=0, freq_std=0.5, phase=True,
                      alpha=(0.2, 1.0) if blend == "alpha" else 1.0,
                      color_max=1.0 if blend == "alpha" else 0.1, depth=(blend == "alpha"))
        cams, vs = None, 0
        cfg_o = oracle_cfg(ora, "2d", H, W, blend, use_rect=True)
        pr = ora.project2d(cfg_o, p)
        kind = "2d"
    else:
        c = gen.make_config(name, seed=0)
        H, W, N, B = c["H"], c["W"], c["N"], c["B"]
        p, cams, vs = c["params"], c["cams"], c["view_stride"]
        cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True)
        pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
        kind = "3d"
    r = gpu_rasterizer(kind, H, W, blend)
    r.forward(to_dev(p), cams, vs)
    torch.cuda.synchronize()
    cand, ell, con = r.render_stats()
    # the kernels' in-ellipse pre-test: e >= log2(alpha_min) - 1e-4 (render.cu make_args)
    thr = cfg_o.alpha_min * 2.0 ** -1e-4
    oc = ora.render_counts(cfg_o, pr, thr)
    ro = ora.render(cfg_o, pr)
    masked = ro["margin"] < 1e-5
    # a masked pixel may stop at another list entry (ALPHA): bound by its list length
    slack_cand = 0
    if blend == "alpha":
        b = ora.bin_sort(cfg_o, pr)
        T = b["tile_offsets"]
        GX, GY = -(-W // 16), -(-H // 16)
        ids = np.nonzero(masked)[0]
        v, rem = ids // (H * W), ids % (H * W)
        t = v * GX * GY + (rem // W) // 16 * GX + (rem % W) // 16
        slack_cand = int((T[t + 1] - T[t]).sum())
    print(f"[counters] {case}: gpu cand {cand} ell {ell} con {con}; oracle cand "
          f"{int(oc['cand'].sum())} ell {int(oc['ell'].sum())} con {int(oc['con'].sum())}; "
          f"masked px {int(masked.sum())}, ambiguous ell pairs {int(oc['amb'].sum())}")
    assert abs(cand - int(oc["cand"].sum())) <= slack_cand
    assert abs(ell - int(oc["ell"].sum())) <= int(oc["amb"].sum()) + slack_cand
    assert abs(con - int(oc["con"].sum())) <= int(masked.sum()) + slack_cand
    if not masked.any():
        assert cand == int(oc["cand"].sum()) and con == int(oc["con"].sum())
    if blend == "sum":
        # SUM candidates are pure integer arithmetic on the CSR offsets
        b = ora.bin_sort(cfg_o, pr)
        T = b["tile_offsets"]
        GX, GY = -(-W // 16), -(-H // 16)
        tot = 0
        for t in range(B * GX * GY):
            tt = t % (GX * GY)
            tx, ty = tt % GX, tt // GX
            npx = (min(W, 16 * tx + 16) - 16 * tx) * (min(H, 16 * ty + 16) - 16 * ty)
            tot += int(T[t + 1] - T[t]) * npx
        assert cand == tot


# ------------------------------------------------- full-size sampled gradients --
@pytest.mark.parametrize("name", ["c3", "c5", "c4"])
def test_full_size_sampled_gradient_parity(ora, name):
    """BASELINE.json configs at full size in the bench's launch configuration
    (C3: 8 x 1080p, 1M primitives, alpha blending; C5: 4K, 3M primitives, SUM —
    its 32400 tiles take the 2-chunk SUM backward; C4: 100 frames of
    1352x1014 (partial tiles on both axes, 85 x 64 grid), 300k per-frame
    primitives, B*T = 544000 so the tile sort takes 3 passes): every integer
    artefact bit-exact, 4096 sampled pixels, and the gradients of a dL/dC
    supported on those pixels (so the oracle's subset gradient is the full
    one), under the exclude-and-count protocol."""
    c = gen.make_config(name, seed=0)
    H, W, N, B = c["H"], c["W"], c["N"], c["B"]
    kind = "2d" if c["kind"] == "2d" else "3d"
    p, cams, vs = c["params"], c["cams"], c["view_stride"]
    cfg_o = oracle_cfg(ora, kind, H, W, c["blend"], use_rect=True)
    pr = ora.project3d(cfg_o, p, cams, view_stride=vs) if kind == "3d" else ora.project2d(cfg_o, p)
    r = gpu_rasterizer(kind, H, W, c["blend"])
    out = r.forward(to_dev(p), cams, vs)
    torch.cuda.synchronize()
    if name == "c4":
        assert B * (-(-W // 16)) * (-(-H // 16)) > 65536  # the 3-pass tile sort
    _check_integers(ora, cfg_o, pr, r, B, N)
    rng = np.random.default_rng(13)
    pix = np.sort(rng.choice(B * H * W, 4096, replace=False))
    dLs = rng.uniform(-1, 1, (4096, 3)).astype(np.float32)
    dLfull = np.zeros((B, 3, H, W), np.float32)
    v, rem = pix // (H * W), pix % (H * W)
    for ch in range(3):
        dLfull[v, ch, rem // W, rem % W] = dLs[:, ch]
    ro = ora.render(cfg_o, pr, pix=pix, dLdC=dLs, abs_terms=True)
    img = _pixels(_np(out["image"]))[pix]
    nbad, namb = pixel_violations(img, ro["color"], ro["margin"])
    assert nbad == 0, (nbad, namb)
    if c["blend"] == "alpha":
        nbad, _ = pixel_violations(_np(out["T_final"]).reshape(-1)[pix], ro["T"], ro["margin"])
        assert nbad == 0
    grads = r.backward(torch.from_numpy(dLfull).cuda())
    torch.cuda.synchronize()
    og, gb = oracle_grads(ora, cfg_o, p, pr, ro, cams, vs)
    exc = ambiguous_rows(pr, ro["margin"], B, N, H, W, view_stride=vs, pix=pix)
    nz = sum(int(np.count_nonzero(np.asarray(v_))) for v_ in og.values())
    assert nz > 1000  # the sample reaches many primitives
    check_grads_strict(grads, og, exc, f"{name} sampled 4096 px", bound=gb)


@pytest.mark.parametrize("case", ["2d_sum", "3d_alpha", "6d_alpha", "3d_sh", "3d_exact"])
def test_chunked_preprocess_backward_bitwise(case):
    """wipes_render_bwd_moments + wipes_preprocess_bwd over parameter-row
    chunks (the bucketed multi-GPU exchange's backward) gives
    bitwise the gradients of the one-shot wipes_render_bwd; every chunk
    callback sees contiguous rows covering all parameter rows once."""
    kw = {}
    if case == "2d_sum":
        H = W = 64
        p = gen.gen2d(H, W, 700, seed=5, freq_std=0.5, phase=True)
        cams, vs, B, kind, blend = None, 0, 1, "2d", "sum"
    else:
        name = "p6d" if case == "6d_alpha" else "p3d"
        over = {"sh_degree": 2} if case == "3d_sh" else {}
        c = gen.make_config(name, seed=0, **over)
        H, W, B = c["H"], c["W"], c["B"]
        p, cams, vs = c["params"], c["cams"], c["view_stride"]
        kind, blend = "3d", "alpha"
        if case == "3d_sh":
            kw["sh_degree"] = 2
        if case == "3d_exact":
            kw["proj"] = "exact"
    dp = to_dev(p)
    dL = torch.from_numpy(gen.gen_dLdC(B, H, W, seed=9)).cuda()
    # deterministic backward: the two passes' moments are bitwise equal, so any
    # difference would come from the row chunking
    r = gpu_rasterizer(kind, H, W, blend, deterministic=1, **kw)
    r.forward(dp, cams, vs)
    ref = {k: v.clone() for k, v in r.backward(dL).items()}
    seen = []
    got = r.backward(dL, row_chunks=3, on_rows=lambda a, b: seen.append((a, b)))
    torch.cuda.synchronize()
    rows = r.grad_rows()
    assert seen[0][0] == 0 and seen[-1][1] == rows and len(seen) == 3
    assert all(a1 == b0 for (_, a1), (b0, _) in zip(seen, seen[1:]))
    for k in ref:
        assert torch.equal(ref[k], got[k]), k


# ------------------------------------------------------------- sort modes --
@pytest.mark.parametrize("mode", ["rts", "onesweep"])
@pytest.mark.parametrize("case", ["c1_sum", "c1_alpha", "p3d", "p6d", "views131"])
def test_sort_modes_integer_parity(ora, case, mode, monkeypatch):
    """Both radix-sort modes (sort.cu) at any size: the run-time threshold
    WIPES_SORT_RTS_TILES = 1 sends every sort through reduce-then-scan (and the
    ALPHA presort through its view-segmented form, segments of one or a few
    ragged tiles), a huge one through onesweep with look-back; keys, values and
    tile ranges stay bit-exact with the oracle and the image within its bound."""
    monkeypatch.setenv("WIPES_SORT_RTS_TILES", "1" if mode == "rts" else str(1 << 40))
    if case.startswith("c1"):
        blend = case.split("_")[1]
        H = W = 64
        N, B = 256, 1
        p = gen.gen2d(H, W, N, seed=0, cov_mode="cholesky", freq_std=0.5, phase=True,
                      alpha=(0.2, 1.0) if blend == "alpha" else 1.0,
                      color_max=1.0 if blend == "alpha" else 0.1, depth=(blend == "alpha"))
        cams, vs, kind = None, 0, "2d"
    elif case == "views131":
        N, B, H, W = 60, 131, 32, 32
        p = gen.gen3d(N, seed=2, scale_mult=20.0)
        cams = [gen.camera((2.5 * np.cos(a), -0.3, 2.5 * np.sin(a)), W, H)
                for a in np.linspace(0, 2 * np.pi, B, endpoint=False)]
        vs, kind, blend = 0, "3d", "alpha"
    else:
        c = gen.make_config(case, seed=0)
        H, W, N, B = c["H"], c["W"], c["N"], c["B"]
        p, cams, vs, kind, blend = c["params"], c["cams"], c["view_stride"], "3d", "alpha"
    if kind == "2d":
        cfg_o = oracle_cfg(ora, "2d", H, W, blend, cov2="cholesky")
        pr = ora.project2d(cfg_o, p)
        r = gpu_rasterizer("2d", H, W, blend, cov2="cholesky")
    else:
        cfg_o = oracle_cfg(ora, "3d", H, W, blend, use_rect=True)
        pr = ora.project3d(cfg_o, p, cams, view_stride=vs)
        r = gpu_rasterizer("3d", H, W, blend)
    out = r.forward(to_dev(p), cams, vs) if kind == "3d" else r.forward(to_dev(p))
    torch.cuda.synchronize()
    _check_integers(ora, cfg_o, pr, r, B, N)
    ro = ora.render(cfg_o, pr)
    nbad, namb = pixel_violations(_pixels(_np(out["image"])), ro["color"], ro["margin"])
    assert nbad == 0, (case, mode, nbad, namb)

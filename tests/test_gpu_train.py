"""GPU parity of the NEXT-2 fitting step (loss, Adam, the fused iteration)
against the oracle's FP64 definitions (tests/test_oracle_train.py pins them).
"""
import numpy as np
import pytest

from paper_2508_12615_b200 import gen
from parity_util import (oracle_cfg, grad_violations, ambiguous_rows, check_grads_strict,
                         oracle_grads)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_12615_b200 import build
    build.build()


def _abi():
    from paper_2508_12615_b200 import abi
    return abi


def _s():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("n", [1, 1000, 3 * 37 * 53, 3 * 512 * 768])
def test_loss_l2_parity_and_determinism(ora, n):
    abi = _abi()
    rng = np.random.default_rng(n)
    a = rng.uniform(0, 1, n).astype(np.float32)
    b = rng.uniform(0, 1, n).astype(np.float32)
    img, tgt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dL = torch.empty_like(img)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    sc = torch.zeros(abi.wipes_train_scratch_bytes(), dtype=torch.uint8, device="cuda")
    for k in range(2):
        abi.check(abi.wipes_loss_l2(img.data_ptr(), tgt.data_ptr(), n, dL.data_ptr(),
                                    loss[k:].data_ptr(), sc.data_ptr(), _s()), "loss")
    torch.cuda.synchronize()
    lo, go = ora.loss_l2(a, b)
    # d = image - target is rounded once to float32 (<= 2^-24 relative)
    assert abs(loss[0].item() - lo) <= 2.5e-7 * lo + 1e-300
    assert loss[0].item() == loss[1].item()  # fixed reduction order
    np.testing.assert_allclose(dL.cpu().numpy(), go, rtol=1e-6, atol=0)


def test_adam_parity_groups_activation_and_guard(ora):
    abi = _abi()
    rng = np.random.default_rng(5)
    sizes, lrs, acts = [7, 1000, 33], [0.05, 2.5e-3, 5e-3], ["none", "none", "sigmoid"]
    P = [rng.normal(size=n).astype(np.float32) for n in sizes]
    M = [np.zeros(n, np.float32) for n in sizes]
    V = [np.zeros(n, np.float32) for n in sizes]
    dev = lambda x: torch.from_numpy(x.copy()).cuda()
    tP, tM, tV = [dev(x) for x in P], [dev(x) for x in M], [dev(x) for x in V]
    tA = [torch.empty_like(x) for x in tP]
    step = torch.zeros(1, dtype=torch.int64, device="cuda")
    guard = torch.zeros(1, dtype=torch.int32, device="cuda")
    sc = torch.zeros(abi.wipes_train_scratch_bytes(), dtype=torch.uint8, device="cuda")
    ref = [dict(p=P[k].astype(np.float64), m=M[k].astype(np.float64), v=V[k].astype(np.float64))
           for k in range(3)]
    for t in range(1, 4):
        G = [rng.normal(size=n).astype(np.float32) for n in sizes]
        tG = [dev(x) for x in G]
        groups = abi.adam_groups([dict(param=tP[k].data_ptr(), grad=tG[k].data_ptr(),
                                       m=tM[k].data_ptr(), v=tV[k].data_ptr(),
                                       act=tA[k].data_ptr() if acts[k] != "none" else None,
                                       n=sizes[k], lr=lrs[k], activation=acts[k])
                                  for k in range(3)])
        abi.check(abi.wipes_adam_step(groups, 3, 0.9, 0.999, 1e-15, step.data_ptr(),
                                      guard.data_ptr(), sc.data_ptr(), _s()), "adam")
        for k in range(3):
            r = ref[k]
            r["p"], r["m"], r["v"], r["a"] = ora.adam_step(r["p"], G[k], r["m"], r["v"], t,
                                                           lrs[k], activation=acts[k])
    torch.cuda.synchronize()
    assert step.item() == 3
    for k in range(3):
        got = tP[k].cpu().numpy()
        tol = 1e-6 * np.abs(ref[k]["p"]) + 1e-3 * lrs[k]
        assert np.all(np.abs(got - ref[k]["p"]) <= tol), k
        if acts[k] == "sigmoid":
            np.testing.assert_allclose(tA[k].cpu().numpy(), ref[k]["a"], rtol=1e-5, atol=1e-7)
    # guard set: nothing moves, the step counter stays
    before = [x.clone() for x in tP]
    guard.fill_(1)
    abi.check(abi.wipes_adam_step(groups, 3, 0.9, 0.999, 1e-15, step.data_ptr(),
                                  guard.data_ptr(), sc.data_ptr(), _s()), "adam")
    torch.cuda.synchronize()
    assert step.item() == 3
    assert all(torch.equal(a, b) for a, b in zip(before, tP))


def _fitter(H, W, N, seed=0, **kw):
    from paper_2508_12615_b200.train import Fitter2D
    tgt = gen.smooth_target(H, W, seed=seed)
    p = gen.init2d_from_target(tgt, N, seed=seed, freq_std=0.1)
    return Fitter2D(torch.from_numpy(tgt).cuda(), {k: torch.from_numpy(v) for k, v in p.items()},
                    **kw), tgt, p


@pytest.mark.parametrize("graph", [False, True])
def test_fit_step_parity(ora, graph):
    """One fused iteration (render -> loss -> backward -> Adam) on C1 sizes
    against the oracle's forward, gradients and Adam step."""
    H = W = 64
    N = 256
    fit, tgt, p = _fitter(H, W, N, graph=graph)
    fit.step()
    torch.cuda.synchronize()
    assert fit.steps_taken() == 1
    # oracle: activated opacity, forward, loss, gradients, Adam (t = 1)
    op = ora.sigmoid(p["opacity"].astype(np.float64)).astype(np.float32)
    q = dict(p, opacity=op)
    cfg = oracle_cfg(ora, "2d", H, W, "sum", cov2="cholesky")
    out = ora.forward(cfg, q)
    img = out["color"].reshape(H, W, 3).transpose(2, 0, 1)
    lo, dL = ora.loss_l2(img, tgt.astype(np.float64))
    assert abs(fit.loss_dev.item() - lo) <= 1e-4 * lo
    ro = ora.render(cfg, out["proj"], dLdC=dL.transpose(1, 2, 0).reshape(-1, 3), abs_terms=True)
    og, gb = oracle_grads(ora, cfg, q, out["proj"], ro)
    from paper_2508_12615_b200.train import DEFAULT_LR
    exc = ambiguous_rows(out["proj"], out["margin"], 1, N, H, W)
    check_grads_strict(fit.grads, og, exc, f"fit step graph={graph}",
                       keys=("mean", "cov", "freq", "color", "opacity"), bound=gb)
    for k in ("mean", "cov", "freq", "color", "opacity"):
        gk = og[k]
        pn, _, _, _ = ora.adam_step(p[k], gk, 0 * gk, 0 * gk, 1, DEFAULT_LR[k],
                                    activation="sigmoid" if k == "opacity" else "none")
        got = fit.raw[k].cpu().numpy()
        sure = np.abs(gk if k != "opacity" else gk * 0.25) > 1e-3 * np.max(np.abs(gk)) + 1e-9
        assert np.allclose(got[sure], pn[sure], rtol=1e-6, atol=1e-4 * DEFAULT_LR[k]), k
        assert np.all(np.abs(got - p[k]) <= DEFAULT_LR[k] * (1 + 1e-5) + 1e-6), k


def test_fit_converges_and_freq_subset_property():
    """Loss falls on a zone plate (128x128, N = 500); with f = 0 and
    lr_f = 0 the frequencies stay exactly 0 (the Gaussian subset)."""
    from paper_2508_12615_b200.train import Fitter2D
    tgt = gen.zone_plate(128, 128, k=60.0)
    p = gen.init2d_from_target(tgt, 500, seed=1, freq_std=0.0)
    tp = {k: torch.from_numpy(v) for k, v in p.items()}
    fit = Fitter2D(torch.from_numpy(tgt).cuda(), tp, lr=dict(freq=0.0))
    l0 = fit.loss()
    hist = fit.fit(300, check_every=100)
    assert fit.steps_taken() == 300
    assert hist[-1][1] < 0.5 * l0, (l0, hist)
    assert torch.count_nonzero(fit.raw["freq"]).item() == 0


def test_fit_overflow_guard_and_recovery():
    """Iterations whose intersections overflow the capacity apply no update;
    fit() grows the workspace and still takes exactly the requested steps."""
    fit, _, _ = _fitter(64, 64, 256, graph=False)
    fit.r._alloc(fit.N, 1, 16)  # shrink the capacity far below the need
    p0 = fit.raw["mean"].clone()
    fit.step()
    torch.cuda.synchronize()
    assert fit.steps_taken() == 0 and torch.equal(p0, fit.raw["mean"])
    fit.fit(5, check_every=2)
    assert fit.steps_taken() == 5
    assert not torch.equal(p0, fit.raw["mean"])


def test_fit_deterministic_loss_curve():
    """same seed + deterministic rasterizer mode => identical loss
    curve and parameters across runs (no float atomics anywhere in the step)."""
    runs = []
    for _ in range(2):
        fit, _, _ = _fitter(64, 64, 256, seed=3, deterministic=1)
        hist = fit.fit(40, check_every=10)
        runs.append((hist, {k: v.clone() for k, v in fit.raw.items()}))
    assert runs[0][0] == runs[1][0]
    for k in runs[0][1]:
        assert torch.equal(runs[0][1][k], runs[1][1][k]), k


def test_fit_alpha_blended_2d_with_depth():
    """NEXT-2's optional 2D alpha-blending mode (a user depth orders
    the primitives; Eq. 3 compositing): the fitting step runs and lowers the loss."""
    from paper_2508_12615_b200.train import Fitter2D
    tgt = gen.smooth_target(64, 64, seed=5)
    p = gen.init2d_from_target(tgt, 300, seed=5, freq_std=0.05)
    p["depth"] = np.random.default_rng(5).uniform(1, 10, 300).astype(np.float32)
    fit = Fitter2D(torch.from_numpy(tgt).cuda(), {k: torch.from_numpy(v) for k, v in p.items()},
                   blend="alpha")
    l0 = fit.loss()
    hist = fit.fit(150, check_every=50)
    assert fit.steps_taken() == 150 and hist[-1][1] < 0.7 * l0, (l0, hist)

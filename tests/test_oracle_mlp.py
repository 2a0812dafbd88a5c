"""Pins of the oracle's NEXT-4 deformation MLP (oracle/mlp.py; PAPER.md:176-180
Eq. 5, Eq. 8). CPU only.

- positional encoding closed forms;
- a hand-computed 2-wide network;
- torch (CPU, float64, nn.Linear + autograd) as an independent
  implementation of the same architecture: outputs and every gradient;
- finite differences of the per-frame deformation (apply, scale exp, frame sums).
"""
import math

import numpy as np
import pytest

from oracle import mlp

torch = pytest.importorskip("torch")


def test_posenc_closed_form():
    g = mlp.posenc(np.zeros((1, 3)), 2)
    np.testing.assert_array_equal(g, [[0, 0, 0, 0, 0, 0, 1, 1, 1, 0, 0, 0, 1, 1, 1]])
    x = np.array([[0.3, -1.2, 2.0]])
    g = mlp.posenc(x, 3)
    assert g.shape == (1, 21)
    np.testing.assert_allclose(g[0, 15:18], np.sin(4 * x[0]))  # k = 2 sine block
    np.testing.assert_allclose(g[0, 18:21], np.cos(4 * x[0]))
    c = mlp.config()
    assert mlp.embed_dim(c) == 63 + 13 == 76


def test_hand_computed_network():
    """width 2, depth 2, skip 0 (layer 1 sees [e, h0]), Lx = Lt = 0: e = (x, t)."""
    c = mlp.config(width=2, depth=2, skip=0, Lx=0, Lt=0)
    assert mlp.embed_dim(c) == 4
    P = {"W0": np.array([[1, 0, 0, 0], [0, -1, 0, 1]], float), "b0": np.array([0.5, 0.0]),
         "W1": np.ones((2, 6)), "b1": np.array([-1.0, 0.0]),
         "Wh": np.zeros((13, 2)), "bh": np.arange(13.0)}
    P["Wh"][0] = [1, 2]
    theta = np.concatenate([P[n].reshape(-1) for n, _, _ in mlp.layout(c)])
    x, t = np.array([[1.0, 2.0, 3.0]]), np.array([0.5])
    out, _ = mlp.forward(c, theta, x, t)
    # e = (1, 2, 3, .5); h0 = relu(1.5, -2 + .5) = (1.5, 0)
    # layer 1 input [e, h0] sums to 8; h1 = relu(8 - 1, 8) = (7, 8); out0 = 7 + 16
    assert out[0, 0] == 23.0
    np.testing.assert_array_equal(out[0, 1:], np.arange(1.0, 13.0))


def _torch_net(c, theta):
    P = mlp.unpack(c, theta)
    layers = []
    for l in range(c["depth"]):
        lin = torch.nn.Linear(mlp.layer_in(c, l), c["width"]).double()
        lin.weight.data = torch.tensor(P[f"W{l}"])
        lin.bias.data = torch.tensor(P[f"b{l}"])
        layers.append(lin)
    head = torch.nn.Linear(c["width"], 13).double()
    head.weight.data = torch.tensor(P["Wh"])
    head.bias.data = torch.tensor(P["bh"])
    return layers, head


def _torch_forward(c, layers, head, e):
    h = e
    for l, lin in enumerate(layers):
        h = torch.relu(lin(h))
        if l == c["skip"]:
            h = torch.cat([e, h], 1)
    return head(h)


@pytest.mark.parametrize("cfg", [dict(width=16, depth=4, skip=1, Lx=3, Lt=2),
                                 dict(width=8, depth=8, skip=4, Lx=10, Lt=6)])
def test_against_torch_autograd(cfg):
    c = mlp.config(**cfg)
    rng = np.random.default_rng(0)
    theta = rng.normal(0, 0.4, mlp.param_count(c))
    x, t = rng.normal(0, 1, (7, 3)), rng.uniform(0, 1, 7)
    out, cache = mlp.forward(c, theta, x, t)
    layers, head = _torch_net(c, theta)
    e = torch.tensor(mlp.embed(c, x, t))
    ref = _torch_forward(c, layers, head, e)
    np.testing.assert_allclose(out, ref.detach().numpy(), rtol=1e-12, atol=1e-12)
    dout = rng.normal(size=out.shape)
    (ref * torch.tensor(dout)).sum().backward()
    g = mlp.unpack(c, mlp.backward(c, theta, cache, dout))
    for l, lin in enumerate(layers):
        np.testing.assert_allclose(g[f"W{l}"], lin.weight.grad.numpy(), rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(g[f"b{l}"], lin.bias.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g["Wh"], head.weight.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g["bh"], head.bias.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_deform_gradients_by_finite_differences():
    c = mlp.config(width=8, depth=3, skip=0, Lx=2, Lt=1)
    rng = np.random.default_rng(2)
    N, times = 4, [0.1, 0.7]
    canon = dict(mean=rng.normal(size=(N, 3)), quat=rng.normal(size=(N, 4)),
                 scale=rng.uniform(0.5, 1.5, (N, 3)), freq=rng.normal(size=(N, 3)))
    theta = rng.normal(0, 0.3, mlp.param_count(c))
    W = {k: rng.normal(size=(len(times) * N, canon[k].shape[1])) for k in canon}

    def loss(th, cn):
        pf, _ = mlp.deform(c, th, cn, times)
        return sum(float(np.sum(pf[k] * W[k])) for k in W)
    pf, cache = mlp.deform(c, theta, canon, times)
    gth, gcn = mlp.deform_backward(c, theta, canon, cache, W)
    h = 1e-6
    for j in rng.choice(theta.size, 25, replace=False):
        tp, tm = theta.copy(), theta.copy()
        tp[j] += h
        tm[j] -= h
        fd = (loss(tp, canon) - loss(tm, canon)) / (2 * h)
        assert abs(fd - gth[j]) <= 1e-6 * max(1.0, abs(fd)), (j, fd, gth[j])
    for k in ("quat", "scale", "freq"):  # mean: stop-gradient into the network (R35)
        for idx in [(0, 0), (N - 1, canon[k].shape[1] - 1)]:
            cp = {a: b.copy() for a, b in canon.items()}
            cm = {a: b.copy() for a, b in canon.items()}
            cp[k][idx] += h
            cm[k][idx] -= h
            fd = (loss(theta, cp) - loss(theta, cm)) / (2 * h)
            assert abs(fd - gcn[k][idx]) <= 1e-6 * max(1.0, abs(fd)), (k, idx)
    # mean: dL/dmu = sum over frames of dL/dmu_t (the network input is stop-gradient)
    np.testing.assert_allclose(gcn["mean"], W["mean"].reshape(2, N, 3).sum(0))


def test_apply_closed_form():
    z = np.zeros((2, 13))
    m, q, s, f = (np.ones((2, 3)), np.ones((2, 4)), np.full((2, 3), 2.0), np.zeros((2, 3)))
    p = mlp.apply(m, q, s, f, z)
    assert np.all(p["mean"] == 1) and np.all(p["scale"] == 2)
    z[:, 7:10] = math.log(3.0)
    np.testing.assert_allclose(mlp.apply(m, q, s, f, z)["scale"], 6.0)


def test_round_bf16():
    """bf16 = the top 16 bits of float32 with round-to-nearest-even."""
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5, 1e-30, 3.0e38])
    r = mlp.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # 1 + 2^-8 is a tie: to the even neighbour 1.0
    assert r[2] == 1.0 + 2 ** -7      # above the tie rounds up
    assert r[3] == -2.5               # exactly representable
    ref = torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(r, ref)

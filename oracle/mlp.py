"""WIPES oracle, NEXT-4 — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The time-conditioned deformation field of PAPER.md Eq. 8:
(dx, df, dSigma) = F_theta(gamma(x), gamma(t)), the D-3DGS network of Eq. 5
 that the paper adopts ("all other ... settings aligned with
D-3DGS"), written out in numpy FP64 from its definition (R34-R36):

  gamma_L(p) = [p, sin(2^0 p), cos(2^0 p), ..., sin(2^(L-1) p), cos(2^(L-1) p)]
  e = [gamma_Lx(x), gamma_Lt(t)]                       (E = 3(1+2Lx) + 1+2Lt)
  h_0 = relu(W_0 e + b_0),  h_l = relu(W_l h_(l-1) + b_l)   l = 1..D-1,
  except the layer after `skip`, whose input is [e, h_skip] (NeRF-style skip)
  out = W_h h_(D-1) + b_h = (dx[3], dq[4], ds[3], df[3])
  mu_t = mu + dx, q_t = q + dq, s_t = s * exp(ds), f_t = f + df;
  x enters the network through a stop-gradient (D-3DGS), so dL/dmu is the
  sum over frames of dL/dmu_t.

Flat parameter layout theta (float): for l = 0..D-1: W_l [W, K_l] row-major,
then b_l [W]; then W_h [13, W], b_h [13]; K_0 = E, K_(skip+1) = E + W, else W.
Pinned by tests/test_oracle_mlp.py (closed forms, a hand-computed example,
torch autograd as an independent implementation, finite differences).
"""
from __future__ import annotations

import numpy as np

NOUT = 13


def config(width=256, depth=8, skip=4, Lx=10, Lt=6):
    return dict(width=width, depth=depth, skip=skip, Lx=Lx, Lt=Lt)


def embed_dim(c) -> int:
    return 3 * (1 + 2 * c["Lx"]) + (1 + 2 * c["Lt"])


def layer_in(c, l) -> int:
    E, W = embed_dim(c), c["width"]
    if l == 0:
        return E
    return E + W if (c["skip"] >= 0 and l == c["skip"] + 1) else W


def layout(c):
    """[(name, shape, offset)] of the flat theta."""
    out, o = [], 0
    W = c["width"]
    for l in range(c["depth"]):
        K = layer_in(c, l)
        out.append((f"W{l}", (W, K), o)); o += W * K
        out.append((f"b{l}", (W,), o)); o += W
    out.append(("Wh", (NOUT, W), o)); o += NOUT * W
    out.append(("bh", (NOUT,), o)); o += NOUT
    return out


def param_count(c) -> int:
    name, shape, o = layout(c)[-1]
    return o + int(np.prod(shape))


def unpack(c, theta):
    th = np.asarray(theta, np.float64)
    return {n: th[o:o + int(np.prod(s))].reshape(s) for n, s, o in layout(c)}


def posenc(p, L):
    """gamma_L(p) row-wise for p [M, d]: [p, sin(2^0 p), cos(2^0 p), ...]."""
    p = np.asarray(p, np.float64)
    parts = [p]
    for k in range(L):
        parts += [np.sin((2.0 ** k) * p), np.cos((2.0 ** k) * p)]
    return np.concatenate(parts, 1)


def embed(c, x, t):
    x = np.asarray(x, np.float64).reshape(-1, 3)
    t = np.asarray(t, np.float64).reshape(-1, 1)
    return np.concatenate([posenc(x, c["Lx"]), posenc(t, c["Lt"])], 1)


def round_bf16(x):
    """Round to the nearest bfloat16 (ties to even), returned as float64: the
    operand precision of the tensor-core kernel (R36)."""
    b = np.ascontiguousarray(np.asarray(x, np.float64).astype(np.float32)).view(np.uint32)
    b = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return b.view(np.float32).astype(np.float64)


def forward(c, theta, x, t, quantize=False):
    """Network outputs [M, 13] and the cache for backward. quantize=True takes
    the kernel's precision decisions (R36): the encoding and every layer's
    activations are rounded to bf16 (so the ReLU masks are decided on the same
    bf16 operands as on the GPU); arithmetic stays FP64."""
    P = unpack(c, theta)
    q = round_bf16 if quantize else (lambda a: a)
    e = q(embed(c, x, t))
    h = e
    ins, hs = [], []
    for l in range(c["depth"]):
        inp = np.concatenate([e, h], 1) if (c["skip"] >= 0 and l == c["skip"] + 1) else h
        ins.append(inp)
        h = q(np.maximum(inp @ P[f"W{l}"].T + P[f"b{l}"], 0.0))
        hs.append(h)
    out = h @ P["Wh"].T + P["bh"]
    return out, dict(e=e, ins=ins, hs=hs)


def backward(c, theta, cache, dout):
    """dL/dtheta (flat) from dL/dout [M, 13] (inputs x, t get no gradient)."""
    P = unpack(c, theta)
    g = {}
    dout = np.asarray(dout, np.float64)
    hs, ins = cache["hs"], cache["ins"]
    g["Wh"] = dout.T @ hs[-1]
    g["bh"] = dout.sum(0)
    dh = dout @ P["Wh"]
    for l in range(c["depth"] - 1, -1, -1):
        dz = dh * (hs[l] > 0)
        g[f"W{l}"] = dz.T @ ins[l]
        g[f"b{l}"] = dz.sum(0)
        if l == 0:
            break
        din = dz @ P[f"W{l}"]
        dh = din[:, embed_dim(c):] if (c["skip"] >= 0 and l == c["skip"] + 1) else din
    flat = np.zeros(param_count(c))
    for n, s, o in layout(c):
        flat[o:o + int(np.prod(s))] = g[n].reshape(-1)
    return flat


def apply(mean, quat, scale, freq, out):
    """Per-frame parameters from the canonical ones and the network output."""
    out = np.asarray(out, np.float64)
    return dict(mean=np.asarray(mean, np.float64) + out[:, 0:3],
                quat=np.asarray(quat, np.float64) + out[:, 3:7],
                scale=np.asarray(scale, np.float64) * np.exp(out[:, 7:10]),
                freq=np.asarray(freq, np.float64) + out[:, 10:13])


def deform(c, theta, canon, times, quantize=False):
    """F frames x N primitives: rows f*N + i. Returns (per-frame params, cache)."""
    N = canon["mean"].shape[0]
    F = len(times)
    x = np.tile(np.asarray(canon["mean"], np.float64), (F, 1))
    t = np.repeat(np.asarray(times, np.float64), N)
    out, cache = forward(c, theta, x, t, quantize=quantize)
    rep = {k: np.tile(np.asarray(canon[k], np.float64), (F, 1) if np.ndim(canon[k]) > 1 else F)
           for k in ("mean", "quat", "scale", "freq")}
    pf = apply(rep["mean"], rep["quat"], rep["scale"], rep["freq"], out)
    cache.update(out=out, N=N, F=F)
    return pf, cache


def deform_backward(c, theta, canon, cache, g_frame):
    """Gradients of the loss w.r.t. theta and the canonical (mean, quat, scale,
    freq) from those w.r.t. the per-frame parameters g_frame [F*N rows]."""
    N, F, out = cache["N"], cache["F"], cache["out"]
    gm = np.asarray(g_frame["mean"], np.float64)
    gq = np.asarray(g_frame["quat"], np.float64)
    gs = np.asarray(g_frame["scale"], np.float64)
    gf = np.asarray(g_frame["freq"], np.float64)
    scale_t = np.tile(np.asarray(canon["scale"], np.float64), (F, 1)) * np.exp(out[:, 7:10])
    dout = np.concatenate([gm, gq, gs * scale_t, gf], 1)
    gtheta = backward(c, theta, cache, dout)

    def fsum(a):
        return a.reshape(F, N, -1).sum(0)
    gcanon = dict(mean=fsum(gm), quat=fsum(gq), scale=fsum(gs * np.exp(out[:, 7:10])),
                  freq=fsum(gf))
    return gtheta, gcanon

"""NEXT-4: the time-conditioned deformation field F_theta (PAPER.md:272-274
Eq. 8; D-3DGS network, Eq. 5) on the tcgen05 tensor cores.

    d = Deformation(N=300_000)                   # D-3DGS shape: 8 x 256, skip 4
    theta = d.init_theta(seed=0)                 # fp32 [param_count]
    frame = d.forward(theta, canon, times)       # per-frame params, rows f*N + i
    ...rasterize(frame, cams, view_stride=N)...
    g_theta, g_canon = d.backward(theta, canon, g_frame)

Every layer runs in libwipes.so (wipes_mlp_forward / wipes_mlp_backward); this
class only owns the buffers. No CPU fallback.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import abi

DEFORMED = ("mean", "quat", "scale", "freq")
COPIED = ("phase", "color", "opacity", "sh")


def _stream():
    return torch.cuda.current_stream().cuda_stream


class Deformation:
    def __init__(self, N: int, width: int = 256, depth: int = 8, skip: int = 4, Lx: int = 10,
                 Lt: int = 6, device="cuda", precision: str = "bf16x3"):
        """precision: "bf16x3" (default) carries every operand as a split-bf16
        pair (~2^-16 relative, near the FP32 D-3DGS network, R38);
        "bf16" single bf16 operands (faster, R36)."""
        if not torch.cuda.is_available():
            raise RuntimeError("Deformation needs a CUDA device (no CPU fallback)")
        abi.lib()
        self.precision = precision
        self.cfg = abi.wipes_mlp_config(width, depth, skip, Lx, Lt, abi.MLP_PRECISION[precision])
        self.P = abi.wipes_mlp_param_count(self.cfg)
        if self.P == 0:
            raise abi.WipesError(abi.WIPES_EINVAL, "wipes_mlp_param_count",
                                 abi.lib().wipes_last_error().decode())
        self.N, self.device = N, torch.device(device)
        self.width, self.depth, self.skip, self.Lx, self.Lt = width, depth, skip, Lx, Lt
        self.ws = None
        self.rows = 0
        self._last = None
        # bumped by every forward: an autograd backward checks it (the
        # workspace holds the activations of one forward only)
        self.generation = 0

    @property
    def embed_dim(self):
        return 3 * (1 + 2 * self.Lx) + 1 + 2 * self.Lt

    def layer_in(self, l):
        if l == 0:
            return self.embed_dim
        return self.embed_dim + self.width if l == self.skip + 1 else self.width

    def init_theta(self, seed: int = 0, head_scale: float = 1.0) -> torch.Tensor:
        """nn.Linear-style init U(-1/sqrt(K), 1/sqrt(K)) for weights and biases
        (host RNG, synthetic: no trained weights exist)."""
        g = np.random.default_rng(seed)
        parts = []
        for l in range(self.depth):
            K = self.layer_in(l)
            b = 1.0 / math.sqrt(K)
            parts += [g.uniform(-b, b, self.width * K), g.uniform(-b, b, self.width)]
        b = head_scale / math.sqrt(self.width)
        parts += [g.uniform(-b, b, 13 * self.width), g.uniform(-b, b, 13)]
        th = np.concatenate(parts).astype(np.float32)
        assert th.size == self.P
        return torch.from_numpy(th).to(self.device)

    def _ensure(self, rows):
        nb = abi.wipes_mlp_workspace_bytes(self.cfg, rows)
        if self.ws is None or self.ws.numel() < nb + 256:
            self.ws = torch.empty(nb + 256, dtype=torch.uint8, device=self.device)
        self.rows, self.ws_bytes = rows, nb

    def _ws_ptr(self):
        p = self.ws.data_ptr()
        return (p + 255) // 256 * 256

    @staticmethod
    def _params(d):
        p = abi.wipes_params()
        for k in DEFORMED + COPIED:
            setattr(p, k, abi.ptr(d.get(k)))
        return p

    def forward(self, theta: torch.Tensor, canon: dict, times, frame: dict = None,
                train: bool = True) -> dict:
        """train=False skips keeping the activations (inference only)."""
        F = len(times)
        rows = self.N * F
        self._ensure(rows)
        if frame is None:
            frame = {k: torch.empty((rows,) + tuple(canon[k].shape[1:]), dtype=torch.float32,
                                    device=self.device)
                     for k in DEFORMED + COPIED if k in canon}
        shc = int(canon["sh"].shape[1]) if "sh" in canon else 0
        cp, fp = self._params(canon), self._params(frame)
        abi.check(abi.wipes_mlp_forward(self.cfg, abi.ptr(theta), self.N, F, list(times), cp, fp,
                                        shc, train, self._ws_ptr(), self.ws_bytes, _stream()),
                  "wipes_mlp_forward")
        self._last = (F, cp, fp, canon, frame, bool(train))
        self.generation += 1
        return frame

    def backward(self, theta: torch.Tensor, canon: dict, g_frame: dict, g_theta=None,
                 g_canon=None):
        if self._last is None:
            raise RuntimeError("Deformation.backward() before forward()")
        F, train = self._last[0], self._last[5]
        if not train:
            raise RuntimeError("Deformation.backward(): the last forward ran with train=False "
                               "and kept no activations")
        if F * self.N != self.rows:
            raise RuntimeError("Deformation.backward(): workspace rows do not match the last "
                               "forward")
        if g_theta is None:
            g_theta = torch.empty(self.P, dtype=torch.float32, device=self.device)
        if g_canon is None:
            g_canon = {k: torch.empty_like(canon[k]) for k in DEFORMED}
        gf, gc = abi.wipes_grads(), abi.wipes_grads()
        for k in DEFORMED:
            setattr(gf, k, abi.ptr(g_frame[k]))
            setattr(gc, k, abi.ptr(g_canon.get(k)))
        abi.check(abi.wipes_mlp_backward(self.cfg, abi.ptr(theta), self.N, F,
                                         self._params(canon), gf, abi.ptr(g_theta), gc,
                                         self._ws_ptr(), self.ws_bytes, _stream()),
                  "wipes_mlp_backward")
        return g_theta, g_canon


class _DeformFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, d: "Deformation", times, keys, theta, *canon_vals):
        canon = {k: v for k, v in zip(keys, canon_vals)}
        frame = d.forward(theta, canon, times, train=True)
        ctx.d, ctx.keys, ctx.canon, ctx.theta = d, keys, canon, theta
        ctx.gen, ctx.F = d.generation, len(times)
        ctx.out_keys = tuple(k for k in DEFORMED + COPIED if k in frame)
        return tuple(frame[k] for k in ctx.out_keys)

    @staticmethod
    def backward(ctx, *g_out):
        if ctx.d.generation != ctx.gen or ctx.d._last[0] != ctx.F:
            raise RuntimeError(
                "deform(): the Deformation ran another forward before this backward; its "
                "workspace holds one forward's activations, so use one Deformation per call "
                f"(generation {ctx.gen}, now {ctx.d.generation})")
        g = dict(zip(ctx.out_keys, g_out))
        g_frame = {k: (g[k] if g.get(k) is not None else torch.zeros_like(ctx.canon[k]).repeat(
            len(g_out[0]) // ctx.canon[k].shape[0], *([1] * (ctx.canon[k].dim() - 1))))
            for k in DEFORMED}
        g_frame = {k: v.contiguous() for k, v in g_frame.items()}
        g_theta, g_canon = ctx.d.backward(ctx.theta, ctx.canon, g_frame)
        grads = []
        F = g_out[0].shape[0] // ctx.canon["mean"].shape[0]
        for k in ctx.keys:
            if k in DEFORMED:
                grads.append(g_canon[k])
            elif g.get(k) is not None:  # copied groups: sum of the frame rows' gradients
                grads.append(g[k].reshape(F, *ctx.canon[k].shape).sum(0))
            else:
                grads.append(None)
        return (None, None, None, g_theta) + tuple(grads)


def deform(d: Deformation, theta: torch.Tensor, canon: dict, times) -> dict:
    """Differentiable deformation: returns the frame rows as a dict; gradients
    flow to theta and the canonical parameters (x enters the network through a
    stop-gradient, R35)."""
    keys = tuple(k for k in DEFORMED + COPIED if k in canon)
    outs = _DeformFn.apply(d, list(times), keys, theta, *[canon[k] for k in keys])
    out_keys = tuple(k for k in DEFORMED + COPIED if k in canon)
    return dict(zip(out_keys, outs))

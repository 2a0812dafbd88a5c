"""NEXT-2: the 2D image-fitting step around the rasterizer.

One iteration (Eq. 4 objective; PAPER.md:299
"all hyperparameters were kept consistent with GSImage"):

    preprocess -> bin_sort -> render_fwd -> wipes_loss_l2 -> render_bwd ->
    wipes_adam_step

Every step is a libwipes.so kernel on the current stream; this module only
owns the buffers (raw parameters, activations, gradients, Adam moments, the
device step counter and loss) and replays the whole iteration as ONE CUDA
graph. The loss stays in device memory; ``fit()`` reads it back every
``check_every`` iterations together with the capacity-overflow word. An
iteration whose intersections overflowed the capacity leaves the parameters,
moments and step counter untouched (device guard in wipes_adam_step), so
``fit()`` grows the workspace, recaptures and carries on: the trajectory is the
one an unbounded capacity would give.

    fit = Fitter2D(target, params, cov2="cholesky")
    fit.fit(1000)
    print(fit.loss(), fit.psnr())
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np
import torch

from . import abi
from .raster import Rasterizer

# Per-group Adam learning rates in the parameters' own units (pixels for mean
# and the covariance factors, rad/px for frequency; R30). The
# frequency rate is the paper's ("learning rate for the frequency
# coefficients" 2.5e-3); the rest are GSImage-lineage proposals.
DEFAULT_LR = dict(mean=0.05, cov=0.02, freq=2.5e-3, phase=5e-3, color=5e-3, opacity=5e-3)
GROUP_ORDER = ("mean", "cov", "freq", "phase", "color", "opacity")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class Fitter2D:
    """Fits ``target`` ([3, H, W] float32 CUDA, values in [0, 1]) with the 2D
    wavelet primitives in ``params`` (raw values: mean, cov (in ``cov2``
    parameterisation), freq, color, opacity_raw [, phase] [, depth]).
    ``opacity`` is passed through a sigmoid ("opacity_raw = 0
    (opacity 0.5)") unless ``opacity_act="none"``."""

    def __init__(self, target: torch.Tensor, params: dict, cov2: str = "cholesky",
                 blend: str = "sum", lr: Optional[dict] = None, betas=(0.9, 0.999),
                 eps: float = 1e-15, opacity_act: str = "sigmoid", graph: bool = True,
                 growth: float = 1.5, **cfg_kw):
        if not torch.cuda.is_available():
            raise RuntimeError("Fitter2D needs a CUDA device (no CPU fallback)")
        if target.dim() != 3 or target.shape[0] != 3:
            raise ValueError("target must be [3, H, W]")
        self.dev = target.device
        self.H, self.W = int(target.shape[1]), int(target.shape[2])
        self.target = target.contiguous().float().unsqueeze(0)
        self.r = Rasterizer(self.W, self.H, prim="2d", blend=blend, cov2=cov2, device=self.dev,
                            growth=growth, **cfg_kw)
        self.lr = dict(DEFAULT_LR, **(lr or {}))
        self.b1, self.b2, self.eps = float(betas[0]), float(betas[1]), float(eps)
        self.raw = {k: v.detach().to(self.dev, torch.float32).contiguous().clone()
                    for k, v in params.items()}
        self.N = int(self.raw["mean"].shape[0])
        self.opacity_act = opacity_act
        self.act = {}
        if opacity_act == "sigmoid":
            self.act["opacity"] = torch.empty_like(self.raw["opacity"])
        self.trainable = [k for k in GROUP_ORDER if k in self.raw]
        self.grads = {k: torch.zeros_like(self.raw[k]) for k in self.trainable}
        self.m = {k: torch.zeros_like(self.raw[k]) for k in self.trainable}
        self.v = {k: torch.zeros_like(self.raw[k]) for k in self.trainable}
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.scratch = torch.zeros(abi.wipes_train_scratch_bytes(), dtype=torch.uint8,
                                   device=self.dev)
        self.image = torch.empty((1, 3, self.H, self.W), dtype=torch.float32, device=self.dev)
        self.T = self.nc = None
        if blend == "alpha":
            self.T = torch.empty((1, self.H, self.W), dtype=torch.float32, device=self.dev)
            self.nc = torch.empty((1, self.H, self.W), dtype=torch.int32, device=self.dev)
        self.dL = torch.zeros_like(self.image)
        self._host = torch.zeros(2, dtype=torch.float64).pin_memory()
        self._groups = abi.adam_groups([
            dict(param=self.raw[k].data_ptr(), grad=self.grads[k].data_ptr(),
                 m=self.m[k].data_ptr(), v=self.v[k].data_ptr(),
                 act=self.act[k].data_ptr() if k in self.act else None,
                 n=self.raw[k].numel(), lr=self.lr[k],
                 activation="sigmoid" if k in self.act else "none")
            for k in self.trainable])
        abi.check(abi.wipes_activate(self._groups, len(self.trainable), _stream()),
                  "wipes_activate")
        self.use_graph = graph
        self.graph = None
        self._size_and_capture()

    # ------------------------------------------------------------ plumbing
    def render_params(self) -> dict:
        p = {k: v for k, v in self.raw.items()}
        for k, v in self.act.items():
            p[k] = v
        return p

    def _iteration(self):
        r = self.r
        r.preprocess(self.render_params(), sync=False)
        r.bin_sort()
        r.render(self.image, self.T, self.nc)
        n = self.image.numel()
        abi.check(abi.wipes_loss_l2(self.image.data_ptr(), self.target.data_ptr(), n,
                                    self.dL.data_ptr(), self.loss_dev.data_ptr(),
                                    self.scratch.data_ptr(), _stream()), "wipes_loss_l2")
        r.backward(self.dL, self.grads)
        guard = abi.wipes_overflow_flag(r._ws_ptr())
        abi.check(abi.wipes_adam_step(self._groups, len(self.trainable), self.b1, self.b2,
                                      self.eps, self.step_dev.data_ptr(), guard,
                                      self.scratch.data_ptr(), _stream()), "wipes_adam_step")

    def _size_and_capture(self):
        # one synced preprocess sizes the intersection capacity (x growth)
        self.r.preprocess(self.render_params(), sync=True)
        torch.cuda.synchronize()
        self.graph = None
        if not self.use_graph:
            return
        # warm the rasterizer kernels once outside capture (no Adam update)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.r.forward(self.render_params(), sync=False)
            self.r.backward(self.dL, self.grads)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._iteration()
        torch.cuda.synchronize()
        self.graph = g
        self._graph_ws = self.r._ws_ptr()

    # ------------------------------------------------------------- public
    def step(self):
        """One iteration, asynchronous (no host sync)."""
        if self.graph is not None:
            if self.r._ws_ptr() != self._graph_ws:  # workspace re-grown outside the graph
                self._size_and_capture()
            self.graph.replay()
        else:
            self._iteration()

    def steps_taken(self) -> int:
        return int(self.step_dev.item())

    def poll(self):
        """(loss of the last iteration, overflowed?) — one small D2H copy."""
        n, o = self.r.check_overflow()
        self._host[0:1].copy_(self.loss_dev, non_blocking=False)
        return float(self._host[0]), bool(o)

    def fit(self, steps: int, check_every: int = 50) -> list:
        """Run until ``steps`` more Adam steps have been applied; returns the
        (step, loss) pairs read at each check."""
        target = self.steps_taken() + steps
        hist = []
        while True:
            done = self.steps_taken()
            if done >= target:
                break
            for _ in range(min(check_every, target - done)):
                self.step()
            loss, overflowed = self.poll()
            if overflowed:  # the overflowed iterations made no update
                self._size_and_capture()
                continue
            if not math.isfinite(loss):
                raise FloatingPointError(f"non-finite loss at step {self.steps_taken()}")
            hist.append((self.steps_taken(), loss))
        return hist

    def loss(self) -> float:
        """L2 loss of the current parameters (one extra forward, no update)."""
        self.r.forward(self.render_params(), sync=True)
        abi.check(abi.wipes_loss_l2(self.r._saved[0].data_ptr(), self.target.data_ptr(),
                                    self.image.numel(), self.dL.data_ptr(),
                                    self.loss_dev.data_ptr(), self.scratch.data_ptr(),
                                    _stream()), "wipes_loss_l2")
        return float(self.loss_dev.item())

    def psnr(self) -> float:
        """PSNR (dB) of the clamped render against the target."""
        img = self.r.forward(self.render_params(), sync=True)["image"].clamp(0, 1)
        mse = float(((img - self.target) ** 2).mean())
        return 99.0 if mse == 0 else min(99.0, 10 * math.log10(1.0 / mse))

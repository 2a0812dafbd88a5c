"""Public Python API of the B200 WIPES rasterizer (thin layer over the C ABI).

    r = Rasterizer(width=768, height=512, prim="2d", blend="sum", cov2="cholesky")
    out = r.forward(params)              # params: dict of CUDA float32 tensors
    grads = r.backward(dL_dimage)        # dict with the same keys as params

or, through autograd, ``image = rasterize(r, params)``.

All compute runs in libwipes.so kernels on the current torch CUDA stream;
torch provides memory, the stream and (in dist.py) process groups only.
Capacity protocol: the first forward reads the intersection
total back once (one sync) and sizes the workspace at 1.25x; later calls are
sync-free and check the device overflow flag only when asked
(``check_overflow()``), re-running the frame if it overflowed.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import abi

PARAM_KEYS_2D = ("mean", "cov", "freq", "phase", "color", "opacity", "depth")
PARAM_KEYS_3D = ("mean", "scale", "quat", "freq", "phase", "color", "opacity", "sh")
GRAD_KEYS = ("mean", "cov", "scale", "quat", "freq", "phase", "color", "opacity", "sh")


def row_ranges(rows: int, chunks: int) -> list:
    """[row0, row1) ranges splitting `rows` into `chunks` contiguous pieces
    (multiples of 64 rows except the last)."""
    chunks = max(1, min(int(chunks), max(1, -(-rows // 64))))
    step = -(-rows // chunks)
    step = -(-step // 64) * 64
    return [(a, min(rows, a + step)) for a in range(0, rows, step)] or [(0, 0)]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _req(t: Optional[torch.Tensor], name: str) -> Optional[torch.Tensor]:
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return t


class Rasterizer:
    def __init__(self, width: int, height: int, prim: str = "2d", blend: str = "sum",
                 cov2: str = "sigma", tile: int = 16, growth: float = 1.25,
                 device: str | torch.device = "cuda", **cfg_kw):
        if not torch.cuda.is_available():
            raise RuntimeError("WIPES rasterizer needs a CUDA device (no CPU fallback)")
        abi.lib()
        self.width, self.height, self.prim, self.blend = width, height, prim, blend
        self.cfg = abi.make_config(width, height, tile=tile, prim=prim, blend=blend, cov2=cov2,
                                   **cfg_kw)
        self.device = torch.device(device)
        self.growth = growth
        self.cap = 0
        self.ws: Optional[torch.Tensor] = None
        self.ws_bytes = 0
        self.N = 0
        self.B = 1
        self._saved = None
        self.n_dup = None
        # forward generation: bumped by every render(); an autograd backward
        # checks it so a second forward before backward raises instead of
        # returning the later frame's gradients (the workspace holds one frame)
        self.generation = 0
        # autograd path: check the device capacity-overflow flag every k
        # backward calls (one stream sync each); 0 disables the check
        self.overflow_check_every = 1
        self._bwd_calls = 0

    # -------------------------------------------------------------- helpers
    @property
    def tiles(self):
        t = self.cfg.tile
        return -(-self.width // t), -(-self.height // t)

    def _alloc(self, N: int, B: int, cap: int):
        nbytes = abi.wipes_workspace_bytes(self.cfg, N, B, cap)
        if nbytes == 0:
            raise abi.WipesError(abi.WIPES_EINVAL, "wipes_workspace_bytes",
                                 abi.lib().wipes_last_error().decode())
        if self.ws is None or self.ws_bytes < nbytes:
            self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            self.ws_bytes = nbytes
        self.cap, self.N, self.B = cap, N, B

    def _ws_ptr(self) -> int:
        p = self.ws.data_ptr()
        return (p + 255) // 256 * 256

    def _params(self, params: dict, view_stride: int):
        keys = PARAM_KEYS_3D if self.prim == "3d" else PARAM_KEYS_2D
        p = abi.wipes_params()
        for k in keys:
            t = _req(params.get(k), k)
            setattr(p, k, abi.ptr(t))
        p.view_stride = int(view_stride)
        return p

    # -------------------------------------------------------------- forward
    def preprocess(self, params: dict, cams=None, view_stride: int = 0, sync: bool = None,
                   cull_flags: Optional[torch.Tensor] = None):
        """Step 1. With sync (default on the first call) reads the intersection
        total back and grows the workspace when needed."""
        mean = params["mean"]
        B = len(cams) if (self.prim == "3d") else 1
        N = int(mean.shape[0]) if (self.prim == "2d" or view_stride == 0) else int(view_stride)
        if self.prim == "3d" and view_stride not in (0, N):
            raise ValueError("view_stride must be 0 or N")
        cp = abi.cameras(cams) if self.prim == "3d" else None
        pp = self._params(params, view_stride)
        if sync is None:
            sync = self.ws is None or self.N != N or self.B != B
        if self.ws is None or self.N != N or self.B != B:
            self._alloc(N, B, max(self.cap, 1024))
        self._keep = (pp, cp, params)
        cf = abi.ptr(cull_flags)
        st, total = abi.wipes_preprocess(self.cfg, pp, N, cp, B, self._ws_ptr(), self.ws_bytes,
                                         self.cap, sync, cf, _stream())
        if st == abi.WIPES_ECAPACITY:
            self._alloc(N, B, max(int(total * self.growth) + 1, 1024))
            st, total = abi.wipes_preprocess(self.cfg, pp, N, cp, B, self._ws_ptr(),
                                             self.ws_bytes, self.cap, True, cf, _stream())
        abi.check(st, "wipes_preprocess")
        if sync:
            self.n_dup = total
        self._cams = cp
        self._pp = pp
        self._view_stride = view_stride
        return self.n_dup

    def bin_sort(self, keys_out=None, vals_out=None, toff_out=None):
        abi.check(abi.wipes_bin_sort(self.cfg, self.N, self.B, self._ws_ptr(), self.ws_bytes,
                                     self.cap, abi.ptr(keys_out), abi.ptr(vals_out),
                                     abi.ptr(toff_out), _stream()), "wipes_bin_sort")

    def render(self, image=None, T_final=None, n_contrib=None):
        B, H, W = self.B, self.height, self.width
        dev = self.device
        if image is None:
            image = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)
        if self.blend == "alpha":
            if T_final is None:
                T_final = torch.empty((B, H, W), dtype=torch.float32, device=dev)
            if n_contrib is None:
                n_contrib = torch.empty((B, H, W), dtype=torch.int32, device=dev)
        abi.check(abi.wipes_render_fwd(self.cfg, self.N, self.B, self._ws_ptr(), self.ws_bytes,
                                       self.cap, abi.ptr(image), abi.ptr(T_final),
                                       abi.ptr(n_contrib), _stream()), "wipes_render_fwd")
        self._saved = (image, T_final, n_contrib)
        self.generation += 1
        return image, T_final, n_contrib

    def forward(self, params: dict, cams=None, view_stride: int = 0, sync: bool = None):
        self.preprocess(params, cams, view_stride, sync=sync)
        self.bin_sort()
        image, T, nc = self.render()
        return dict(image=image, T_final=T, n_contrib=nc)

    def check_overflow(self):
        st, n, o = abi.wipes_check_overflow(self._ws_ptr(), self.ws_bytes, _stream())
        abi.check(st, "wipes_check_overflow")
        return n, bool(o)

    # ------------------------------------------------------------- backward
    def backward(self, dL_dimage: torch.Tensor, grads: Optional[dict] = None,
                 row_chunks: int = 1, on_rows=None) -> dict:
        """Gradients of every parameter group. row_chunks > 1 splits the
        preprocess backward into that many parameter-row ranges (one launch
        each, wipes_preprocess_bwd) and calls on_rows(row0, row1) after each is
        enqueued on the current stream: a multi-GPU caller starts the
        all-reduce of rows [row0, row1) there, overlapping the next chunk
        (dist.GradBucket.reduce_rows)."""
        if self._saved is None:
            raise RuntimeError("backward() before forward()")
        _req(dL_dimage, "dL_dimage")
        pp, cp, params = self._keep
        _, T, nc = self._saved
        if grads is None:
            grads = {}
            for k in GRAD_KEYS:
                t = params.get(k)
                if t is not None:
                    grads[k] = torch.empty_like(t)
        g = abi.wipes_grads()
        for k in GRAD_KEYS:
            setattr(g, k, abi.ptr(grads.get(k)))
        if row_chunks <= 1 and on_rows is None:
            abi.check(abi.wipes_render_bwd(self.cfg, pp, self.N, cp, self.B, self._ws_ptr(),
                                           self.ws_bytes, self.cap, abi.ptr(dL_dimage),
                                           abi.ptr(T), abi.ptr(nc), g, _stream()),
                      "wipes_render_bwd")
            return grads
        abi.check(abi.wipes_render_bwd_moments(self.cfg, self.N, self.B, self._ws_ptr(),
                                               self.ws_bytes, self.cap, abi.ptr(dL_dimage),
                                               abi.ptr(T), abi.ptr(nc), _stream()),
                  "wipes_render_bwd_moments")
        rows = self.grad_rows()
        for r0, r1 in row_ranges(rows, row_chunks):
            abi.check(abi.wipes_preprocess_bwd(self.cfg, pp, self.N, cp, self.B, self._ws_ptr(),
                                               self.ws_bytes, self.cap, g, r0, r1, _stream()),
                      "wipes_preprocess_bwd")
            if on_rows is not None:
                on_rows(r0, r1)
        return grads

    def grad_rows(self) -> int:
        """Parameter-gradient rows: primitives (2D or a shared 3D set) or
        (view, primitive) rows of per-frame sets."""
        return self.N if (self.prim == "2d" or self._view_stride == 0) else self.B * self.N

    # ----------------------------------------------------------- debug/parity
    def get_preprocess(self):
        BN = self.B * self.N
        dev = self.device
        out = dict(rect=torch.empty((BN, 4), dtype=torch.int32, device=dev),
                   count=torch.empty(BN, dtype=torch.int32, device=dev),
                   offsets=torch.empty(BN, dtype=torch.int64, device=dev),
                   depth_key=torch.empty(BN, dtype=torch.int32, device=dev),
                   records=torch.empty((BN, 16), dtype=torch.float32, device=dev))
        abi.check(abi.wipes_get_preprocess(self.cfg, self.N, self.B, self._ws_ptr(),
                                           self.ws_bytes, self.cap, abi.ptr(out["rect"]),
                                           abi.ptr(out["count"]), abi.ptr(out["offsets"]),
                                           abi.ptr(out["depth_key"]), abi.ptr(out["records"]),
                                           _stream()), "wipes_get_preprocess")
        return out

    def render_stats(self):
        """(tile-method candidate pairs, in-ellipse pairs, contributing pairs)
        of the current frame (measurement only)."""
        out = torch.zeros(3, dtype=torch.int64, device=self.device)
        abi.check(abi.wipes_render_stats(self.cfg, self.N, self.B, self._ws_ptr(), self.ws_bytes,
                                         self.cap, abi.ptr(out), _stream()), "wipes_render_stats")
        return tuple(int(x) for x in out.cpu())

    def get_grad_moments(self):
        out = torch.empty((self.B * self.N, abi.GRAD_MOMENTS), dtype=torch.float32,
                          device=self.device)
        abi.check(abi.wipes_get_grad_moments(self.cfg, self.N, self.B, self._ws_ptr(),
                                             self.ws_bytes, self.cap, abi.ptr(out), _stream()),
                  "wipes_get_grad_moments")
        return out

    def bin_sort_outputs(self):
        """Re-run bin_sort with copies of keys, values and tile offsets."""
        n, _ = self.check_overflow()
        gx, gy = self.tiles
        dev = self.device
        keys = torch.empty(max(self.cap, 1), dtype=torch.int64, device=dev)
        vals = torch.empty(max(self.cap, 1), dtype=torch.int32, device=dev)
        toff = torch.empty(self.B * gx * gy + 1, dtype=torch.int32, device=dev)
        self.bin_sort(keys, vals, toff)
        return keys[:n], vals[:n], toff


class CapacityOverflow(RuntimeError):
    """The frame's tile intersections exceeded the workspace capacity, so its
    image and gradients were truncated (SURVEY §8(b) capacity protocol). The
    capacity has been grown; re-run the step."""


class _RasterizeFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, r: Rasterizer, cams, view_stride, keys, *tensors):
        params = {k: t for k, t in zip(keys, tensors) if t is not None}
        out = r.forward(params, cams=cams, view_stride=view_stride)
        ctx.r, ctx.keys, ctx.gen = r, keys, r.generation
        return out["image"]

    @staticmethod
    def backward(ctx, g):
        r = ctx.r
        if r.generation != ctx.gen:
            raise RuntimeError(
                "rasterize(): the Rasterizer ran another forward before this backward; its "
                "workspace holds one frame, so use one Rasterizer per frame in a loss "
                f"(forward generation {ctx.gen}, now {r.generation})")
        r._bwd_calls += 1
        k = r.overflow_check_every
        if k and r._bwd_calls % k == 0:
            n, over = r.check_overflow()
            if over:
                r._alloc(r.N, r.B, int(n * r.growth) + 1)
                r.generation += 1  # the truncated frame is gone
                raise CapacityOverflow(
                    f"rasterize(): {n} tile intersections exceeded the capacity; the frame was "
                    f"truncated. Capacity grown to {r.cap}: re-run the step.")
        grads = r.backward(g.contiguous())
        return (None, None, None, None) + tuple(grads.get(k) for k in ctx.keys)


def rasterize(r: Rasterizer, params: dict, cams=None, view_stride: int = 0) -> torch.Tensor:
    """Differentiable render: returns image [B,3,H,W]; gradients flow to params."""
    keys = tuple(k for k in (PARAM_KEYS_3D if r.prim == "3d" else PARAM_KEYS_2D) if k in params)
    return _RasterizeFn.apply(r, cams, view_stride, keys, *[params[k] for k in keys])


class FrameGraph:
    """CUDA-graph capture of one frame of a Rasterizer on fixed device buffers.

    The forward (preprocess -> bin_sort -> render) and the backward (render
    backward -> preprocess backward [-> optional hook, e.g. a gradient
    all_reduce]) are captured as two graphs and replayed with ``forward()`` /
    ``backward()``: no host work or host sync per frame. The intersection
    capacity is sized by one synced forward before capture (x growth); if the
    parameters later change so much that the capacity overflows,
    ``check_overflow()`` reports it and ``recapture()`` re-sizes.
    """

    def __init__(self, r: Rasterizer, params: dict, cams=None, view_stride: int = 0,
                 dL_dimage: Optional[torch.Tensor] = None, grads: Optional[dict] = None,
                 backward_hook=None):
        self.r, self.params, self.cams, self.vs = r, params, cams, view_stride
        self.dL, self.grads, self.hook = dL_dimage, grads, backward_hook
        self.recapture()

    def recapture(self):
        r = self.r
        r.forward(self.params, self.cams, self.vs, sync=True)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm the captured path once on a side stream
            self._fwd()
            if self.dL is not None:
                self._bwd()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.g_fwd = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_fwd):
            self._fwd()
        self.g_bwd = None
        if self.dL is not None:
            self.g_bwd = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_bwd):
                self._bwd()
        torch.cuda.synchronize()

    def _fwd(self):
        r = self.r
        r.preprocess(self.params, self.cams, self.vs, sync=False)
        r.bin_sort()
        img, T, nc = r._saved if r._saved is not None else (None, None, None)
        self.out = r.render(img, T, nc)

    def _bwd(self):
        self.grads = self.r.backward(self.dL, self.grads)
        if self.hook is not None:
            self.hook(self.grads)

    def forward(self):
        self.g_fwd.replay()
        return self.out

    def backward(self):
        self.g_bwd.replay()
        return self.grads

    def step(self):
        self.g_fwd.replay()
        if self.g_bwd is not None:
            self.g_bwd.replay()

    def check_overflow(self):
        return self.r.check_overflow()

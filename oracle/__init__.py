"""WIPES oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, double-precision CPU implementation of the WIPES rasterizer
(arXiv 2508.12615) used to prove the CUDA path correct. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product package
``paper_2508_12615_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.cpp`` (see its header for the paper
passages each function follows); this module only builds it with gcc
(``-O2 -fopenmp -ffp-contract=off -fno-fast-math``) and marshals numpy arrays.

Parity status: pinned by ``tests/test_oracle_*.py`` (closed forms, invariants,
finite differences, DFT, brute-force compositing). The exact z-integration
mode (``exact_proj=1``) is pinned by 1-D quadrature of its kernel value, its
chain rule by whole-pipeline finite differences and by agreement with the
paper-mode chain at f = 0. The NEXT-2 fitting step (``loss_l2``,
``adam_step``, ``sigmoid``) is written out below in numpy FP64 from its
textbook definitions and pinned by closed forms in tests/test_oracle_train.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-std=c++17"]


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *GCC_FLAGS, _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class ora_cfg(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tile", C.c_int32),
                ("prim3d", C.c_int32), ("alpha_blend", C.c_int32), ("cov2", C.c_int32),
                ("extent", C.c_int32), ("ewa_clamp", C.c_int32), ("exact_proj", C.c_int32),
                ("use_rect", C.c_int32),
                ("alpha_min", C.c_double), ("alpha_max", C.c_double), ("T_min", C.c_double),
                ("dilation", C.c_double), ("cov_eps", C.c_double), ("det_min", C.c_double),
                ("bg", C.c_double * 3), ("color_per_view", C.c_int32)]


class ora_cam(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("near_z", C.c_double), ("far_z", C.c_double)]


COV_MODES = {"sigma": 0, "cholesky": 1, "rs": 2}


@dataclass
class Cfg:
    """Oracle configuration. Constants are float32-rounded where the CUDA path
    receives float32 (so both sides decide with the same threshold values)."""
    width: int
    height: int
    tile: int = 16
    prim3d: bool = False
    alpha_blend: bool = False
    cov2: str = "sigma"
    extent: str = "opacity"      # or "sigma3"
    ewa_clamp: bool = True
    exact_proj: bool = False
    use_rect: bool = False
    alpha_min: float = float(np.float32(1.0 / 255.0))
    alpha_max: float = float(np.float32(0.99))
    T_min: float = float(np.float32(1e-4))
    dilation: float = 0.0
    cov_eps: float = 0.0
    det_min: float = float(np.float32(1e-12))
    bg: tuple = (0.0, 0.0, 0.0)
    sh_degree: Optional[int] = None  # NEXT-3: None = flat RGB `color`; 0..3 = SH `sh`

    def c(self, color_per_view: bool = False) -> ora_cfg:
        return ora_cfg(self.width, self.height, self.tile, int(self.prim3d),
                       int(self.alpha_blend), COV_MODES[self.cov2],
                       0 if self.extent == "opacity" else 1, int(self.ewa_clamp),
                       int(self.exact_proj), int(self.use_rect),
                       self.alpha_min, self.alpha_max, self.T_min, self.dilation,
                       self.cov_eps, self.det_min, (C.c_double * 3)(*self.bg),
                       int(color_per_view))


P_FIELDS = ["mux", "muy", "a", "b", "c", "fx", "fy", "phi", "beta", "cr", "cg", "cb",
            "alpha", "depth", "sxx", "sxy", "syy", "rmargin", "rx", "ry"]
G_FIELDS = ["mux", "muy", "a", "b", "c", "fx", "fy", "phi", "beta", "cr", "cg", "cb", "alpha"]
NP_ = len(P_FIELDS)
NG_ = len(G_FIELDS)

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.ora_bin.restype = C.c_int64
        assert _lib.ora_record_width() == NP_ and _lib.ora_grad_width() == NG_
    return _lib


def _d(a):
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def cams_c(cams):
    arr = (ora_cam * len(cams))()
    for k, cm in enumerate(cams):
        arr[k].R = (C.c_double * 9)(*np.asarray(cm["R"], np.float64).reshape(9))
        arr[k].t = (C.c_double * 3)(*np.asarray(cm["t"], np.float64).reshape(3))
        for nm in ("fx", "fy", "cx", "cy"):
            setattr(arr[k], nm, float(cm[nm]))
        arr[k].near_z = float(cm.get("near", 0.01))
        arr[k].far_z = float(cm.get("far", 100.0))
    return arr


@dataclass
class Projected:
    N: int
    B: int
    flag: np.ndarray
    rect: np.ndarray
    count: np.ndarray
    keylo: np.ndarray
    rec: np.ndarray

    def field(self, name):
        return self.rec[:, P_FIELDS.index(name)]


def project2d(cfg: Cfg, p: dict) -> Projected:
    """O1 — 2D preprocess of parameter dict p (mean, cov, freq, [phase], color,
    opacity, [depth])."""
    N = int(np.asarray(p["mean"]).shape[0])
    mean, cov, freq = _d(p["mean"]), _d(p["cov"]), _d(p["freq"])
    phase, color, op = _d(p.get("phase")), _d(p["color"]), _d(p["opacity"])
    depth = _d(p.get("depth"))
    flag = np.zeros(N, np.int32)
    rect = np.zeros((N, 4), np.int32)
    count = np.zeros(N, np.int32)
    keylo = np.zeros(N, np.uint32)
    rec = np.zeros((N, NP_), np.float64)
    cf = cfg.c()
    lib().ora_project2d(C.byref(cf), C.c_int64(N), _p(mean), _p(cov), _p(freq), _p(phase),
                        _p(color), _p(op), _p(depth), _p(flag), _p(rect), _p(count),
                        _p(keylo), _p(rec))
    return Projected(N, 1, flag, rect, count, keylo, rec)


def project3d(cfg: Cfg, p: dict, cams, view_stride: int = 0) -> Projected:
    """O2 — 3D preprocess for B cameras. view_stride (in primitives): 0 = one
    shared parameter set, N = per-view parameter sets (6D)."""
    B = len(cams)
    mean = _d(p["mean"]).reshape(-1, 3)
    N = mean.shape[0] if view_stride == 0 else int(view_stride)
    scale, quat, freq = _d(p["scale"]), _d(p["quat"]), _d(p["freq"])
    phase, op = _d(p.get("phase")), _d(p["opacity"])
    cc = cams_c(cams)
    if cfg.sh_degree is not None:  # NEXT-3: per (view, primitive) SH colours
        color = sh_colors(cfg.sh_degree, mean, p["sh"], cams, N, view_stride)
    else:
        color = _d(p["color"])
    flag = np.zeros(B * N, np.int32)
    rect = np.zeros((B * N, 4), np.int32)
    count = np.zeros(B * N, np.int32)
    keylo = np.zeros(B * N, np.uint32)
    rec = np.zeros((B * N, NP_), np.float64)
    cf = cfg.c(color_per_view=cfg.sh_degree is not None)
    lib().ora_project3d(C.byref(cf), C.c_int64(N), C.c_int32(B), cc, _p(mean), _p(scale),
                        _p(quat), _p(freq), _p(phase), _p(color), _p(op),
                        C.c_int64(view_stride), _p(flag), _p(rect), _p(count), _p(keylo),
                        _p(rec))
    return Projected(N, B, flag, rect, count, keylo, rec)


def bin_sort(cfg: Cfg, pr: Projected):
    """O6 — offsets, sorted (key, value) pairs and per-tile CSR offsets."""
    B, N = pr.B, pr.N
    GX = -(-cfg.width // cfg.tile)
    GY = -(-cfg.height // cfg.tile)
    offsets = np.zeros(B * N, np.int64)
    total = int(lib().ora_bin(C.byref(cfg.c()), C.c_int64(N), C.c_int32(B), _p(pr.rect),
                              _p(pr.count), _p(pr.keylo), _p(offsets), None, None, None,
                              C.c_int64(0)))
    keys = np.zeros(max(total, 1), np.uint64)
    vals = np.zeros(max(total, 1), np.uint32)
    toff = np.zeros(B * GX * GY + 1, np.int64)
    lib().ora_bin(C.byref(cfg.c()), C.c_int64(N), C.c_int32(B), _p(pr.rect), _p(pr.count),
                  _p(pr.keylo), _p(offsets), _p(keys), _p(vals), _p(toff),
                  C.c_int64(total))
    return dict(offsets=offsets, keys=keys[:total], vals=vals[:total], tile_offsets=toff,
                total=total)


def render(cfg: Cfg, pr: Projected, pix=None, dLdC=None, nthreads: int = 0,
           abs_terms: bool = False):
    """O3-O5 — brute-force render of the listed pixels (flat ids v*H*W+y*W+x;
    None = all pixels of all views). Returns dict(color [npix,3], T, margin,
    ncomp, rgrad [B*N, 13] if dLdC given (dLdC is [npix, 3])); with abs_terms
    also rgrad_abs [B*N, 13], the sum over pairs of the absolute values of every
    term of each record gradient (the running error bound scale, R23b)."""
    B, N = pr.B, pr.N
    if pix is not None:
        pix = np.ascontiguousarray(np.asarray(pix, np.int64))
        npix = pix.shape[0]
    else:
        npix = B * cfg.height * cfg.width
    color = np.zeros((npix, 3), np.float64)
    T = np.zeros(npix, np.float64)
    margin = np.zeros(npix, np.float64)
    ncomp = np.zeros(npix, np.int32)
    rgrad = rgrad_abs = None
    if dLdC is not None:
        dLdC = _d(dLdC).reshape(npix, 3)
        rgrad = np.zeros((B * N, NG_), np.float64)
        if abs_terms:
            rgrad_abs = np.zeros((B * N, NG_), np.float64)
    rec = np.ascontiguousarray(pr.rec)
    lib().ora_render(C.byref(cfg.c()), C.c_int64(N), C.c_int32(B), _p(rec), _p(pr.flag),
                     _p(pr.rect), _p(pr.keylo), C.c_int64(npix), _p(pix), _p(color), _p(T),
                     _p(margin), _p(ncomp), _p(dLdC), _p(rgrad), C.c_int32(nthreads),
                     _p(rgrad_abs))
    return dict(color=color, T=T, margin=margin, ncomp=ncomp, rgrad=rgrad, rgrad_abs=rgrad_abs)


def render_counts(cfg: Cfg, pr: Projected, thr_ell: float):
    """Roofline work counters per pixel over its tile list (oracle.cpp
    ora_render_counts): dict(cand, ell, con, amb) of int64 [B*H*W]."""
    B, N = pr.B, pr.N
    n = B * cfg.height * cfg.width
    out = {k: np.zeros(n, np.int64) for k in ("cand", "ell", "con", "amb")}
    rec = np.ascontiguousarray(pr.rec)
    lib().ora_render_counts(C.byref(cfg.c()), C.c_int64(N), C.c_int32(B), _p(rec),
                            _p(pr.flag), _p(pr.rect), _p(pr.keylo), C.c_double(thr_ell),
                            _p(out["cand"]), _p(out["ell"]), _p(out["con"]), _p(out["amb"]))
    return out


def image_pixels_to_planar(color, B, H, W):
    """[B*H*W, 3] -> [B, 3, H, W]"""
    return np.ascontiguousarray(color.reshape(B, H, W, 3).transpose(0, 3, 1, 2))


def planar_to_pixels(img):
    """[B, 3, H, W] -> [B*H*W, 3]"""
    img = np.asarray(img)
    return np.ascontiguousarray(img.transpose(0, 2, 3, 1).reshape(-1, 3))


def chain2d(cfg: Cfg, p: dict, pr: Projected, rgrad):
    N = pr.N
    out = {k: np.zeros(s, np.float64) for k, s in
           [("mean", (N, 2)), ("cov", (N, 3)), ("freq", (N, 2)), ("phase", (N,)),
            ("color", (N, 3)), ("opacity", (N,))]}
    lib().ora_chain2d(C.byref(cfg.c()), C.c_int64(N), _p(_d(p["cov"])), _p(pr.flag),
                      _p(np.ascontiguousarray(pr.rec)), _p(_d(rgrad)), _p(out["mean"]),
                      _p(out["cov"]), _p(out["freq"]), _p(out["phase"]), _p(out["color"]),
                      _p(out["opacity"]))
    return out


def chain3d(cfg: Cfg, p: dict, cams, pr: Projected, rgrad, view_stride: int = 0):
    """3D chain rule. Paper mode: analytic (oracle.cpp ora_chain3d); exact mode:
    J^T g with J the central-difference Jacobian of the exact projection."""
    N, B = pr.N, pr.B
    NP = N if view_stride == 0 else B * N
    out = {k: np.zeros(s, np.float64) for k, s in
           [("mean", (NP, 3)), ("scale", (NP, 3)), ("quat", (NP, 4)), ("freq", (NP, 3)),
            ("phase", (NP,)), ("color", (NP, 3)), ("opacity", (NP,))]}
    fn = lib().ora_chain3d_exact if cfg.exact_proj else lib().ora_chain3d
    fn(C.byref(cfg.c()), C.c_int64(N), C.c_int32(B), cams_c(cams),
                      _p(_d(p["mean"])), _p(_d(p["scale"])), _p(_d(p["quat"])),
                      _p(_d(p["freq"])), _p(pr.flag), _p(np.ascontiguousarray(pr.rec)),
                      _p(_d(rgrad)), C.c_int64(view_stride), _p(out["mean"]),
                      _p(out["scale"]), _p(out["quat"]), _p(out["freq"]), _p(out["phase"]),
                      _p(out["color"]), _p(out["opacity"]))
    if cfg.sh_degree is not None:  # colour comes from SH: dL/dsh + view-direction term
        K = (cfg.sh_degree + 1) ** 2
        del out["color"]
        out["sh"] = np.zeros((NP, K, 3), np.float64)
        lib().ora_sh_chain(C.c_int32(cfg.sh_degree), C.c_int64(N), C.c_int32(B), cams_c(cams),
                           _p(_d(p["mean"])), _p(_d(p["sh"])), C.c_int64(view_stride),
                           _p(pr.flag), _p(_d(rgrad)), _p(out["sh"]), _p(out["mean"]))
    return out


def grad_bound(cfg: Cfg, p: dict, pr: Projected, rgrad_abs, cams=None, view_stride: int = 0):
    """Per parameter-gradient element, sum_{v,q} |J_vq| S_vq: the record-
    gradient abs-term scales S = rgrad_abs (render(..., abs_terms=True)) carried
    through the chain rule with every (view, record component) taken apart and
    in absolute value. The chain is linear in the record gradients, so one call
    per (view, component) with that component alone gives its exact signed
    contribution. Returns a dict shaped like chain2d / chain3d."""
    B, N = pr.B, pr.N
    sep_views = cfg.prim3d and view_stride == 0 and B > 1  # rows sum over views
    out = None
    for v in (range(B) if sep_views else [None]):
        for q in range(NG_):
            r = np.zeros_like(rgrad_abs)
            sl = slice(None) if v is None else slice(v * N, (v + 1) * N)
            r[sl, q] = rgrad_abs[sl, q]
            if not np.any(r[:, q]):
                continue
            g = chain3d(cfg, p, cams, pr, r, view_stride) if cfg.prim3d else chain2d(cfg, p, pr, r)
            if out is None:
                out = {k: np.abs(x) for k, x in g.items()}
            else:
                for k in out:
                    out[k] += np.abs(g[k])
    if out is None:
        g = chain3d(cfg, p, cams, pr, rgrad_abs * 0, view_stride) if cfg.prim3d else \
            chain2d(cfg, p, pr, rgrad_abs * 0)
        out = {k: np.abs(x) for k, x in g.items()}
    return out


def sh_basis(deg: int, dirs) -> np.ndarray:
    """O9: real SH basis values [n, (deg+1)^2] at unit directions [n, 3]."""
    d = _d(dirs).reshape(-1, 3)
    K = (deg + 1) ** 2
    out = np.zeros((d.shape[0], K), np.float64)
    lib().ora_sh_basis(C.c_int32(deg), C.c_int64(d.shape[0]), _p(d), _p(out))
    return out


def sh_colors(deg: int, mean, sh, cams, N: int, view_stride: int = 0) -> np.ndarray:
    """O9: SH colour of every (view, primitive) [B*N, 3] (clamped at 0)."""
    B = len(cams)
    out = np.zeros((B * N, 3), np.float64)
    lib().ora_sh_colors(C.c_int32(deg), C.c_int64(N), C.c_int32(B), cams_c(cams),
                        _p(_d(mean)), _p(_d(sh)), C.c_int64(view_stride), _p(out))
    return out


# ---- small scalar helpers (wrappers of the C kernel evaluators) ------------
def eval_wavelet2(conic, f, phi, beta, dx, dy) -> float:
    L = lib()
    L.ora_eval_wavelet2.restype = C.c_double
    c = (C.c_double * 3)(*conic)
    ff = (C.c_double * 2)(*f)
    return L.ora_eval_wavelet2(c, ff, C.c_double(phi), C.c_double(beta), C.c_double(dx),
                               C.c_double(dy))


def eval_gaussian2(conic, dx, dy) -> float:
    L = lib()
    L.ora_eval_gaussian2.restype = C.c_double
    c = (C.c_double * 3)(*conic)
    return L.ora_eval_gaussian2(c, C.c_double(dx), C.c_double(dy))


def eval_wavelet3(inv_cov, f, phi, beta, d) -> float:
    L = lib()
    L.ora_eval_wavelet3.restype = C.c_double
    ic = (C.c_double * 9)(*np.asarray(inv_cov, np.float64).reshape(9))
    ff = (C.c_double * 3)(*f)
    dd = (C.c_double * 3)(*d)
    return L.ora_eval_wavelet3(ic, ff, C.c_double(phi), C.c_double(beta), dd)


def cov2d(mode: str, params) -> np.ndarray:
    out = np.zeros(3, np.float64)
    pp = _d(params)
    lib().ora_cov2d(C.c_int32(COV_MODES[mode]), _p(pp), _p(out))
    return out


# ---- whole-pipeline conveniences used by tests and the CPU baseline --------
def forward(cfg: Cfg, p: dict, cams=None, view_stride=0, pix=None, dLdC=None, nthreads=0):
    pr = project3d(cfg, p, cams, view_stride) if cfg.prim3d else project2d(cfg, p)
    out = render(cfg, pr, pix=pix, dLdC=dLdC, nthreads=nthreads)
    out["proj"] = pr
    return out


def forward_backward(cfg: Cfg, p: dict, dLdC, cams=None, view_stride=0, pix=None,
                     nthreads=0):
    out = forward(cfg, p, cams, view_stride, pix=pix, dLdC=dLdC, nthreads=nthreads)
    pr = out["proj"]
    if cfg.prim3d:
        out["grads"] = chain3d(cfg, p, cams, pr, out["rgrad"], view_stride)
    else:
        out["grads"] = chain2d(cfg, p, pr, out["rgrad"])
    return out


# ---------------------------------------------------------------------------
# NEXT-2: the fitting step around the rasterizer. Plain
# numpy FP64, definitions written out.
# ---------------------------------------------------------------------------
def loss_l2(image, target):
    """L2 loss, mean over pixels and channels, and its gradient
    dL/dimage = 2 (image - target) / n."""
    d = np.asarray(image, np.float64) - np.asarray(target, np.float64)
    n = d.size
    return float(np.sum(d * d) / n), 2.0 * d / n


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))


def adam_step(param, grad, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-15, activation="none"):
    """Adam (Kingma & Ba 2015, Alg. 1; SPEC S:321-324 AdamState defaults) at
    step t >= 1 on the raw parameter; ``grad`` is dL/d(act(param)) and is
    chained through the activation first. Returns (param, m, v, act)."""
    p = np.asarray(param, np.float64)
    g = np.asarray(grad, np.float64)
    if activation == "sigmoid":
        s = sigmoid(p)
        g = g * s * (1.0 - s)
    m = b1 * np.asarray(m, np.float64) + (1.0 - b1) * g
    v = b2 * np.asarray(v, np.float64) + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    p = p - lr * mh / (np.sqrt(vh) + eps)
    act = sigmoid(p) if activation == "sigmoid" else p
    return p, m, v, act

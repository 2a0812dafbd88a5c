"""Thin ctypes binding of libwipes.so (include/wipes.h) — argument marshalling only.

Every step of the rasterizer runs in the CUDA kernels behind these calls;
PyTorch only supplies device memory, the current stream and process groups.
There is NO CPU fallback: if libwipes.so is missing or no CUDA device is
present, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# WIPES_LIB overrides the library path (kernel-variant experiments only)
LIB_PATH = os.environ.get("WIPES_LIB") or os.path.join(_HERE, "libwipes.so")

WIPES_OK, WIPES_EINVAL, WIPES_ECAPACITY, WIPES_ECUDA, WIPES_EUNSUPPORTED = range(5)
PRIM = {"2d": 0, "3d": 1}
BLEND = {"sum": 0, "alpha": 1}
COV2 = {"sigma": 0, "cholesky": 1, "rs": 2}
PROJ = {"paper": 0, "exact": 1}
EXTENT = {"opacity": 0, "sigma3": 1}
COLOR = {"rgb": 0, "sh": 1}
GRAD_MOMENTS = 12
MAX_CAMS_PER_LAUNCH = 128


class wipes_camera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float),
                ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("near_z", C.c_float), ("far_z", C.c_float)]


class wipes_config(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tile", C.c_int32),
                ("prim", C.c_int32), ("blend", C.c_int32), ("cov2", C.c_int32),
                ("proj", C.c_int32), ("extent", C.c_int32),
                ("alpha_min", C.c_float), ("alpha_max", C.c_float), ("T_min", C.c_float),
                ("dilation", C.c_float), ("cov_eps", C.c_float), ("det_min", C.c_float),
                ("ewa_clamp", C.c_int32), ("background", C.c_float * 3),
                ("deterministic", C.c_int32), ("row_mod", C.c_int32), ("row_rem", C.c_int32),
                ("color_mode", C.c_int32), ("sh_degree", C.c_int32),
                ("grad_accum", C.c_int32)]


class wipes_params(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("mean", "cov", "scale", "quat", "freq", "phase",
                                          "color", "opacity", "depth")] + \
               [("view_stride", C.c_int64), ("sh", C.c_void_p)]


class wipes_grads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("mean", "cov", "scale", "quat", "freq", "phase",
                                          "color", "opacity", "sh")]


class wipes_adam_group(C.Structure):
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("m", C.c_void_p),
                ("v", C.c_void_p), ("act", C.c_void_p), ("n", C.c_int64), ("lr", C.c_float),
                ("activation", C.c_int32)]


class wipes_gemm_args(C.Structure):
    _fields_ = [("A", C.c_void_p), ("B", C.c_void_p), ("C", C.c_void_p), ("bias", C.c_void_p),
                ("mask", C.c_void_p), ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
                ("lda", C.c_int64), ("ldb", C.c_int64), ("ldc", C.c_int64), ("ldm", C.c_int64),
                ("a_mn_major", C.c_int32), ("b_mn_major", C.c_int32), ("epilogue", C.c_int32),
                ("split_k", C.c_int32), ("colsum", C.c_void_p), ("split3", C.c_int64)]


class wipes_mlp_config(C.Structure):
    _fields_ = [("width", C.c_int32), ("depth", C.c_int32), ("skip", C.c_int32),
                ("Lx", C.c_int32), ("Lt", C.c_int32), ("precision", C.c_int32)]


MLP_PRECISION = {"bf16x3": 0, "bf16": 1}


GEMM_EPI = {"store_f32": 0, "bias_f32": 1, "bias_relu_bf16": 2, "mask_bf16": 3,
            "atomic_f32": 4}

ACT = {"none": 0, "sigmoid": 1}
MAX_ADAM_GROUPS = 8


class WipesError(RuntimeError):
    def __init__(self, status, where, detail):
        super().__init__(f"{where}: {status_name(status)}: {detail}")
        self.status = status


_lib = None


def lib():
    """Load libwipes.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libwipes.so not built at {LIB_PATH}: run "
                           "`python -m paper_2508_12615_b200.build` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
    P = C.POINTER
    L.wipes_workspace_bytes.argtypes = [P(wipes_config), i64, i32, i64]
    L.wipes_workspace_bytes.restype = sz
    L.wipes_preprocess.argtypes = [P(wipes_config), P(wipes_params), i64, P(wipes_camera), i32,
                                   vp, sz, i64, P(C.c_int64), vp, vp]
    L.wipes_bin_sort.argtypes = [P(wipes_config), i64, i32, vp, sz, i64, vp, vp, vp, vp]
    L.wipes_check_overflow.argtypes = [vp, sz, P(C.c_int64), P(C.c_int32), vp]
    L.wipes_get_preprocess.argtypes = [P(wipes_config), i64, i32, vp, sz, i64, vp, vp, vp, vp,
                                       vp, vp]
    L.wipes_render_fwd.argtypes = [P(wipes_config), i64, i32, vp, sz, i64, vp, vp, vp, vp]
    L.wipes_render_bwd.argtypes = [P(wipes_config), P(wipes_params), i64, P(wipes_camera), i32,
                                   vp, sz, i64, vp, vp, vp, P(wipes_grads), vp]
    L.wipes_render_bwd_moments.argtypes = [P(wipes_config), i64, i32, vp, sz, i64, vp, vp, vp,
                                           vp]
    L.wipes_preprocess_bwd.argtypes = [P(wipes_config), P(wipes_params), i64, P(wipes_camera),
                                       i32, vp, sz, i64, P(wipes_grads), i64, i64, vp]
    L.wipes_get_grad_moments.argtypes = [P(wipes_config), i64, i32, vp, sz, i64, vp, vp]
    L.wipes_render_stats.argtypes = [P(wipes_config), i64, i32, vp, sz, i64, vp, vp]
    L.wipes_train_scratch_bytes.restype = sz
    L.wipes_loss_l2.argtypes = [vp, vp, i64, vp, vp, vp, vp]
    L.wipes_adam_step.argtypes = [P(wipes_adam_group), i32, C.c_float, C.c_float, C.c_float, vp,
                                  vp, vp, vp]
    L.wipes_activate.argtypes = [P(wipes_adam_group), i32, vp]
    L.wipes_overflow_flag.argtypes = [vp]
    L.wipes_overflow_flag.restype = vp
    L.wipes_mlp_param_count.argtypes = [P(wipes_mlp_config)]
    L.wipes_mlp_param_count.restype = sz
    L.wipes_mlp_workspace_bytes.argtypes = [P(wipes_mlp_config), i64]
    L.wipes_mlp_workspace_bytes.restype = sz
    L.wipes_mlp_forward.argtypes = [P(wipes_mlp_config), vp, i64, i32, P(C.c_float),
                                    P(wipes_params), P(wipes_params), i32, i32, vp, sz, vp]
    L.wipes_mlp_forward.restype = C.c_int
    L.wipes_mlp_backward.argtypes = [P(wipes_mlp_config), vp, i64, i32, P(wipes_params),
                                     P(wipes_grads), vp, P(wipes_grads), vp, sz, vp]
    L.wipes_mlp_backward.restype = C.c_int
    L.wipes_gemm_bf16.argtypes = [P(wipes_gemm_args), vp]
    L.wipes_gemm_bf16.restype = C.c_int
    L.wipes_num_kernels.restype = C.c_int
    L.wipes_kernel_name.argtypes = [C.c_int]
    L.wipes_kernel_name.restype = C.c_char_p
    L.wipes_timing_enable.argtypes = [C.c_int]
    L.wipes_timing_collect.argtypes = [P(C.c_double), P(C.c_int64), C.c_int]
    L.wipes_launch_count.restype = C.c_int64
    L.wipes_status_string.argtypes = [C.c_int]
    L.wipes_status_string.restype = C.c_char_p
    L.wipes_last_error.restype = C.c_char_p
    L.wipes_abi_version.restype = C.c_int
    for fn in ("wipes_preprocess", "wipes_bin_sort", "wipes_check_overflow",
               "wipes_get_preprocess", "wipes_render_fwd", "wipes_render_bwd",
               "wipes_render_bwd_moments", "wipes_preprocess_bwd",
               "wipes_get_grad_moments", "wipes_timing_collect", "wipes_render_stats",
               "wipes_loss_l2", "wipes_adam_step", "wipes_activate"):
        getattr(L, fn).restype = C.c_int
    _lib = L
    return L


EXPORTED = ["wipes_workspace_bytes", "wipes_preprocess", "wipes_bin_sort",
            "wipes_check_overflow", "wipes_get_preprocess", "wipes_render_fwd",
            "wipes_render_bwd", "wipes_render_bwd_moments", "wipes_preprocess_bwd",
            "wipes_get_grad_moments", "wipes_render_stats",
            "wipes_train_scratch_bytes", "wipes_loss_l2", "wipes_adam_step", "wipes_activate",
            "wipes_overflow_flag", "wipes_gemm_bf16", "wipes_mlp_param_count",
            "wipes_mlp_workspace_bytes", "wipes_mlp_forward", "wipes_mlp_backward",
            "wipes_num_kernels",
            "wipes_kernel_name", "wipes_timing_enable", "wipes_timing_collect",
            "wipes_launch_count", "wipes_status_string", "wipes_last_error",
            "wipes_abi_version"]


def status_name(s: int) -> str:
    return lib().wipes_status_string(s).decode()


def check(status: int, where: str):
    if status != WIPES_OK:
        raise WipesError(status, where, lib().wipes_last_error().decode())


ACCUM = {"auto": 0, "f32": 1, "f64": 2}


def make_config(width, height, tile=16, prim="2d", blend="sum", cov2="sigma", proj="paper",
                extent="opacity", alpha_min=1.0 / 255.0, alpha_max=0.99, T_min=1e-4,
                dilation=None, cov_eps=0.0, det_min=1e-12, ewa_clamp=True,
                background=(0.0, 0.0, 0.0), deterministic=0, row_mod=0,
                row_rem=0, sh_degree=None, grad_accum="auto") -> wipes_config:
    """sh_degree None: flat RGB `color`; 0..3: SH colour from `sh` (3D, NEXT-3).
    grad_accum: render-backward moment precision, "auto" (FP64 for 3D, FP32 for
    2D), "f32" or "f64" (include/wipes.h WIPES_ACCUM_*, R37)."""
    if dilation is None:
        dilation = 0.3 if prim == "3d" else 0.0
    return wipes_config(int(width), int(height), int(tile), PRIM[prim], BLEND[blend], COV2[cov2],
                        PROJ[proj], EXTENT[extent], alpha_min, alpha_max, T_min, dilation,
                        cov_eps, det_min, int(bool(ewa_clamp)), (C.c_float * 3)(*background),
                        int(deterministic), int(row_mod), int(row_rem),
                        COLOR["rgb"] if sh_degree is None else COLOR["sh"],
                        0 if sh_degree is None else int(sh_degree), ACCUM[grad_accum])


def cameras(cams) -> "C.Array":
    arr = (wipes_camera * max(len(cams), 1))()
    for k, cm in enumerate(cams):
        R = [float(x) for x in list(_flat(cm["R"]))]
        t = [float(x) for x in list(_flat(cm["t"]))]
        arr[k].R = (C.c_float * 9)(*R)
        arr[k].t = (C.c_float * 3)(*t)
        arr[k].fx, arr[k].fy = float(cm["fx"]), float(cm["fy"])
        arr[k].cx, arr[k].cy = float(cm["cx"]), float(cm["cy"])
        arr[k].near_z = float(cm.get("near", 0.01))
        arr[k].far_z = float(cm.get("far", 100.0))
    return arr


def _flat(x):
    try:
        import numpy as np
        return np.asarray(x, dtype=np.float64).reshape(-1)
    except Exception:  # pragma: no cover
        return x


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


# ---- same-name wrappers: marshalling only --------------------------------
def wipes_workspace_bytes(cfg, N, B, cap) -> int:
    return int(lib().wipes_workspace_bytes(C.byref(cfg), N, B, cap))


def wipes_preprocess(cfg, params, N, cams, B, ws, ws_bytes, cap, n_dup_out, cull_flags, stream):
    n = C.c_int64(0)
    st = lib().wipes_preprocess(C.byref(cfg), C.byref(params), N,
                                cams if cams is not None else None, B, ws, ws_bytes, cap,
                                C.byref(n) if n_dup_out else None, cull_flags, stream)
    return st, n.value


def wipes_bin_sort(cfg, N, B, ws, ws_bytes, cap, keys_out, vals_out, toff_out, stream):
    return lib().wipes_bin_sort(C.byref(cfg), N, B, ws, ws_bytes, cap, keys_out, vals_out,
                                toff_out, stream)


def wipes_check_overflow(ws, ws_bytes, stream):
    n, o = C.c_int64(0), C.c_int32(0)
    st = lib().wipes_check_overflow(ws, ws_bytes, C.byref(n), C.byref(o), stream)
    return st, n.value, o.value


def wipes_get_preprocess(cfg, N, B, ws, ws_bytes, cap, rect, count, offsets, dkey, records,
                         stream):
    return lib().wipes_get_preprocess(C.byref(cfg), N, B, ws, ws_bytes, cap, rect, count,
                                      offsets, dkey, records, stream)


def wipes_render_fwd(cfg, N, B, ws, ws_bytes, cap, image, T_final, n_contrib, stream):
    return lib().wipes_render_fwd(C.byref(cfg), N, B, ws, ws_bytes, cap, image, T_final,
                                  n_contrib, stream)


def wipes_render_bwd(cfg, params, N, cams, B, ws, ws_bytes, cap, dLdC, T_final, n_contrib,
                     grads, stream):
    return lib().wipes_render_bwd(C.byref(cfg), C.byref(params), N,
                                  cams if cams is not None else None, B, ws, ws_bytes, cap,
                                  dLdC, T_final, n_contrib, C.byref(grads), stream)


def wipes_render_bwd_moments(cfg, N, B, ws, ws_bytes, cap, dLdC, T_final, n_contrib, stream):
    return lib().wipes_render_bwd_moments(C.byref(cfg), N, B, ws, ws_bytes, cap, dLdC, T_final,
                                          n_contrib, stream)


def wipes_preprocess_bwd(cfg, params, N, cams, B, ws, ws_bytes, cap, grads, row0, row1, stream):
    return lib().wipes_preprocess_bwd(C.byref(cfg), C.byref(params), N,
                                      cams if cams is not None else None, B, ws, ws_bytes, cap,
                                      C.byref(grads), row0, row1, stream)


def wipes_get_grad_moments(cfg, N, B, ws, ws_bytes, cap, out, stream):
    return lib().wipes_get_grad_moments(C.byref(cfg), N, B, ws, ws_bytes, cap, out, stream)


def wipes_render_stats(cfg, N, B, ws, ws_bytes, cap, stats3, stream):
    return lib().wipes_render_stats(C.byref(cfg), N, B, ws, ws_bytes, cap, stats3, stream)


def wipes_train_scratch_bytes() -> int:
    return int(lib().wipes_train_scratch_bytes())


def wipes_loss_l2(image, target, n, dL_dimage, loss, scratch, stream):
    return lib().wipes_loss_l2(image, target, n, dL_dimage, loss, scratch, stream)


def adam_groups(groups):
    """list of dicts (param, grad, m, v, act, n, lr, activation) -> ctypes array."""
    arr = (wipes_adam_group * max(len(groups), 1))()
    for k, g in enumerate(groups):
        arr[k] = wipes_adam_group(g["param"], g["grad"], g["m"], g["v"], g.get("act"), g["n"],
                                  float(g["lr"]), ACT[g.get("activation", "none")])
    return arr


def wipes_adam_step(groups, n_groups, beta1, beta2, eps, step, guard, scratch, stream):
    return lib().wipes_adam_step(groups, n_groups, beta1, beta2, eps, step, guard, scratch,
                                 stream)


def wipes_activate(groups, n_groups, stream):
    return lib().wipes_activate(groups, n_groups, stream)


def wipes_overflow_flag(ws) -> int:
    return int(lib().wipes_overflow_flag(ws) or 0)


def wipes_gemm_bf16(args, stream):
    return lib().wipes_gemm_bf16(C.byref(args), stream)


def gemm(A, B, C, M, N, K, lda, ldb, ldc, epilogue="store_f32", a_mn=False, b_mn=False,
         bias=None, mask=None, ldm=0, split_k=1, colsum=None, stream=None):
    """Marshal a wipes_gemm_args from torch tensors / ints and launch."""
    g = wipes_gemm_args(ptr(A), ptr(B), ptr(C), ptr(bias), ptr(mask), M, N, K, lda, ldb, ldc,
                        ldm, int(a_mn), int(b_mn), GEMM_EPI[epilogue], split_k, ptr(colsum))
    check(wipes_gemm_bf16(g, stream), "wipes_gemm_bf16")


def wipes_mlp_param_count(cfg) -> int:
    return int(lib().wipes_mlp_param_count(C.byref(cfg)))


def wipes_mlp_workspace_bytes(cfg, rows) -> int:
    return int(lib().wipes_mlp_workspace_bytes(C.byref(cfg), rows))


def wipes_mlp_forward(cfg, theta, N, F, times, canon, frame, sh_coeffs, train, ws, ws_bytes,
                      stream):
    t = (C.c_float * max(F, 1))(*[float(x) for x in times])
    return lib().wipes_mlp_forward(C.byref(cfg), theta, N, F, t, C.byref(canon), C.byref(frame),
                                   sh_coeffs, int(train), ws, ws_bytes, stream)


def wipes_mlp_backward(cfg, theta, N, F, canon, g_frame, g_theta, g_canon, ws, ws_bytes, stream):
    return lib().wipes_mlp_backward(C.byref(cfg), theta, N, F, C.byref(canon), C.byref(g_frame),
                                    g_theta, C.byref(g_canon), ws, ws_bytes, stream)


def kernel_names():
    L = lib()
    return [L.wipes_kernel_name(k).decode() for k in range(L.wipes_num_kernels())]


def timing_enable(on: bool):
    lib().wipes_timing_enable(1 if on else 0)


def timing_collect():
    L = lib()
    n = L.wipes_num_kernels()
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    check(L.wipes_timing_collect(ms, cnt, n), "wipes_timing_collect")
    names = kernel_names()
    return {names[k]: (ms[k], cnt[k]) for k in range(n)}


def launch_count() -> int:
    return int(lib().wipes_launch_count())

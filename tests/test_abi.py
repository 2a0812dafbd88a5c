"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/wipes.h declares, and validates arguments BEFORE any launch
(no compute calls — there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

from paper_2508_12615_b200 import abi, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return abi.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "wipes.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wipes_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(abi.EXPORTED)


def test_abi_version_and_strings(L):
    assert L.wipes_abi_version() == 4
    assert abi.status_name(abi.WIPES_EINVAL) == "WIPES_EINVAL"
    assert "render_fwd" in abi.kernel_names()


def test_workspace_bytes_monotone(L):
    cfg = abi.make_config(768, 512)
    a = abi.wipes_workspace_bytes(cfg, 70000, 1, 100000)
    b = abi.wipes_workspace_bytes(cfg, 70000, 1, 400000)
    assert 0 < a < b
    bad = abi.make_config(768, 512, tile=12)
    assert abi.wipes_workspace_bytes(bad, 10, 1, 10) == 0


def _pp():
    p = abi.wipes_params()
    for k in ("mean", "cov", "freq", "color", "opacity"):
        setattr(p, k, 0x1000)
    return p


@pytest.mark.parametrize("mut,msg", [
    (dict(tile=12), "tile"),
    (dict(width=0), "width"),
    (dict(width=20000), "width"),
    (dict(alpha_min=0.5, alpha_max=0.4), "alpha"),
])
def test_einval_before_launch(L, mut, msg):
    kw = dict(width=64, height=64)
    kw.update(mut)
    cfg = abi.make_config(**kw)
    st, _ = abi.wipes_preprocess(cfg, _pp(), 10, None, 1, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL
    assert msg in L.wipes_last_error().decode()


def test_einval_null_and_alignment(L):
    cfg = abi.make_config(64, 64)
    p = _pp()
    p.cov = None
    st, _ = abi.wipes_preprocess(cfg, p, 10, None, 1, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"cov" in L.wipes_last_error()
    p = _pp()
    p.mean = 0x1002
    st, _ = abi.wipes_preprocess(cfg, p, 10, None, 1, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"misaligned" in L.wipes_last_error()
    st, _ = abi.wipes_preprocess(cfg, _pp(), 10, None, 1, 0x100010, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"256-byte" in L.wipes_last_error()
    st, _ = abi.wipes_preprocess(cfg, _pp(), 10, None, 1, 0x100000, 16, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"ws_bytes" in L.wipes_last_error()
    # 2D needs B == 1; 3D needs cameras
    st, _ = abi.wipes_preprocess(cfg, _pp(), 10, None, 2, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL
    cfg3 = abi.make_config(64, 64, prim="3d")
    p3 = _pp()
    p3.scale = 0x1000
    p3.quat = 0x1000
    st, _ = abi.wipes_preprocess(cfg3, p3, 10, None, 1, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"cams" in L.wipes_last_error()


def test_bad_modes(L):
    cfg = abi.make_config(64, 64, prim="2d", deterministic=2)
    st, _ = abi.wipes_preprocess(cfg, _pp(), 10, None, 1, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"deterministic" in L.wipes_last_error()
    cfg = abi.make_config(64, 64, prim="2d", sh_degree=2)
    st, _ = abi.wipes_preprocess(cfg, _pp(), 10, None, 1, 0x100000, 1 << 30, 100, False, None, None)
    assert st == abi.WIPES_EINVAL and b"SH" in L.wipes_last_error()


def test_deterministic_workspace_has_slots(L):
    c0 = abi.make_config(64, 64)
    c1 = abi.make_config(64, 64, deterministic=1)
    n0 = abi.wipes_workspace_bytes(c0, 1000, 1, 10000)
    n1 = abi.wipes_workspace_bytes(c1, 1000, 1, 10000)
    assert n1 - n0 >= 10000 * (4 + 2 * 48)  # prevals + 2 footprints x 12 floats per dup


def test_exact_projection_workspace_has_beta_moments(L):
    """NEXT-1: the exact mode adds one float per (view, primitive) record."""
    c0 = abi.make_config(64, 64, prim="3d")
    c1 = abi.make_config(64, 64, prim="3d", proj="exact")
    n0 = abi.wipes_workspace_bytes(c0, 100000, 2, 0)
    n1 = abi.wipes_workspace_bytes(c1, 100000, 2, 0)
    assert n1 - n0 >= 4 * 200000


def test_product_package_never_imports_oracle():
    """The product path must not import, call or link the oracle."""
    pkg = os.path.join(ROOT, "paper_2508_12615_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                s = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\bimport\s+oracle\b|from\s+oracle\b|oracle\.cpp|liboracle",
                                     s), f


def test_train_entry_points_validate(L):
    """NEXT-2 entry points reject bad arguments before any launch."""
    assert abi.wipes_train_scratch_bytes() >= 8 * 1184
    st = abi.wipes_loss_l2(0x1000, 0x2000, 10, None, 0x3000, 0x4000, None)
    assert st == abi.WIPES_EINVAL
    st = abi.wipes_loss_l2(0x1000, 0x2000, 10, 0x1000, 0x3000, 0x4000, None)
    assert st == abi.WIPES_EINVAL and b"alias" in L.wipes_last_error()
    g = abi.adam_groups([dict(param=0x1000, grad=0x2000, m=0x3000, v=0x4000, n=4, lr=0.1,
                              activation="sigmoid")])
    st = abi.wipes_adam_step(g, 1, 0.9, 0.999, 1e-15, 0x5000, None, 0x6000, None)
    assert st == abi.WIPES_EINVAL and b"act" in L.wipes_last_error()
    g = abi.adam_groups([dict(param=0x1000, grad=0x2000, m=0x3000, v=0x4000, n=4, lr=0.1)])
    st = abi.wipes_adam_step(g, 1, 1.0, 0.999, 1e-15, 0x5000, None, 0x6000, None)
    assert st == abi.WIPES_EINVAL and b"beta" in L.wipes_last_error()
    st = abi.wipes_adam_step(g, 9, 0.9, 0.999, 1e-15, 0x5000, None, 0x6000, None)
    assert st == abi.WIPES_EINVAL
    assert abi.wipes_overflow_flag(0x100000) == 0x100000 + 8

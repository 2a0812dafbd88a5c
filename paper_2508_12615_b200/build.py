"""Build libwipes.so (sm_100a) in-tree with nvcc.

preprocess.cu is compiled with --fmad=false: its FP64 expressions must round
exactly as written (pinned order) so tile rects match the oracle
bit for bit. The render kernels keep FMA contraction (they use explicit
__fmaf_rn / __fmul_rn anyway).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libwipes.so")
BUILD = os.path.join(ROOT, "build", "wipes")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          f"-I{os.path.join(ROOT, 'include')}"]
SOURCES = {
    "preprocess.cu": ["--fmad=false"],
    "preprocess_bwd.cu": [],
    "binning.cu": [],
    "sort.cu": [],
    "render.cu": [],
    "train.cu": [],
    "gemm.cu": [],
    "gemm_e0.cu": [],
    "gemm_e1.cu": [],
    "gemm_e2.cu": [],
    "gemm_e3.cu": [],
    "gemm_e4.cu": [],
    "mlp.cu": [],
    "mlp_fused.cu": [],
    "abi.cu": [],
}


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every .cu for sm_100a and link libwipes.so. `defines`/`out`
    build an experimental variant elsewhere: with defines and no `out`, the
    variant goes to libwipes_<defines>.so beside the in-tree library, which a
    variant build never touches (load it with WIPES_LIB=...)."""
    tag = "_".join(d.replace("=", "") for d in defines)
    if defines and out is None:
        out = os.path.join(HERE, f"libwipes_{tag}.so")
    if defines and os.path.abspath(out) == os.path.abspath(LIB):
        raise ValueError("a build with defines must not overwrite the in-tree libwipes.so")
    lib = out or LIB
    bdir = BUILD if not defines else BUILD + "_" + tag
    os.makedirs(bdir, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "wipes.h")]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    def compile_one(item):
        src, extra = item
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [_nvcc(), *ARCH, *COMMON, *extra, *[f"-D{d}" for d in defines], "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r

    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES.items()))
    objs = []
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else None))

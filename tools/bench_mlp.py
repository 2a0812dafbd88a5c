"""NEXT-4 measurement: deformation MLP forward + backward (tcgen05) at the C4
primitive count, timed with CUDA events; per-GEMM breakdown via the library's
kernel timing. Usage: python tools/bench_mlp.py [N] [F]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_12615_b200 import abi, gen  # noqa: E402
from paper_2508_12615_b200.deform import Deformation  # noqa: E402


def flops_per_row(d):
    f = 0
    for l in range(d.depth):
        K = d.layer_in(l)
        f += 2 * d.width * K
    f += 2 * 13 * d.width
    return f


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    d = Deformation(N)
    theta = d.init_theta(0, head_scale=0.1)
    p = gen.gen3d(N, seed=0)
    canon = {k: torch.from_numpy(v).cuda() for k, v in p.items()}
    times = list(np.linspace(0, 1, F))
    frame = d.forward(theta, canon, times)
    g = {k: torch.randn_like(frame[k]) for k in ("mean", "quat", "scale", "freq")}
    d.backward(theta, canon, g)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    res = {}
    for name, fn in (("fwd", lambda: d.forward(theta, canon, times, frame)),
                     ("bwd", lambda: d.backward(theta, canon, g))):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(10):
            fn()
        b.record(s)
        b.synchronize()
        res[name] = a.elapsed_time(b) / 10
    abi.timing_enable(True)
    d.forward(theta, canon, times, frame)
    d.backward(theta, canon, g)
    torch.cuda.synchronize()
    abi.timing_enable(False)
    kt = {k: round(v[0], 4) for k, v in abi.timing_collect().items() if v[1]}
    rows = N * F
    fr = flops_per_row(d)
    fwd_fl = rows * fr
    bwd_fl = rows * (2 * fr - 2 * d.width * d.layer_in(0))  # dW for all + dIn except layer 0
    out = dict(N=N, F=F, fwd_ms=res["fwd"], bwd_ms=res["bwd"],
               fwd_tflops=fwd_fl / res["fwd"] / 1e9, bwd_tflops=bwd_fl / res["bwd"] / 1e9,
               kernel_ms=kt)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

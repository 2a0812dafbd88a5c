"""Micro-benchmark of the tcgen05 GEMM (NEXT-4 building block): one shape,
every operand-major combination and epilogue, CUDA-event timed."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_12615_b200 import abi  # noqa: E402


def main():
    M, N, K = 300000, 256, 256
    dev = "cuda"
    A = torch.randn(M, K, device=dev).to(torch.bfloat16)
    At = A.t().contiguous()
    W = torch.randn(N, K, device=dev).to(torch.bfloat16)
    Wt = W.t().contiguous()
    bias = torch.randn(N, device=dev)
    mask = torch.randn(M, N, device=dev).to(torch.bfloat16)
    Cb = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    Cf = torch.empty(M, N, device=dev)
    cs = torch.zeros(N, device=dev)
    s = torch.cuda.current_stream()
    res = {}
    cases = {
        "KK_bias_relu": dict(A=A, B=W, C=Cb, lda=K, ldb=K, epilogue="bias_relu_bf16", bias=bias),
        "KM_bias_relu": dict(A=A, B=Wt, C=Cb, lda=K, ldb=N, b_mn=True, epilogue="bias_relu_bf16", bias=bias),
        "KK_mask": dict(A=A, B=W, C=Cb, lda=K, ldb=K, epilogue="mask_bf16", mask=mask, ldm=N),
        "KM_mask": dict(A=A, B=Wt, C=Cb, lda=K, ldb=N, b_mn=True, epilogue="mask_bf16", mask=mask, ldm=N),
        "KM_mask_colsum": dict(A=A, B=Wt, C=Cb, lda=K, ldb=N, b_mn=True, epilogue="mask_bf16", mask=mask, ldm=N, colsum=cs),
        "KK_store_f32": dict(A=A, B=W, C=Cf, lda=K, ldb=K, epilogue="store_f32"),
        "MK_bias_relu": dict(A=At, B=W, C=Cb, lda=M, ldb=K, a_mn=True, epilogue="bias_relu_bf16", bias=bias),
    }
    for name, kw in cases.items():
        C = kw.pop("C")
        args = dict(kw)
        fn = lambda: abi.gemm(args["A"], args["B"], C, M, N, K, args["lda"], args["ldb"], N,
                              epilogue=args["epilogue"], a_mn=args.get("a_mn", False),
                              b_mn=args.get("b_mn", False), bias=args.get("bias"),
                              mask=args.get("mask"), ldm=args.get("ldm", 0),
                              colsum=args.get("colsum"))
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            fn()
        b.record(s)
        b.synchronize()
        ms = a.elapsed_time(b) / 20
        res[name] = dict(us=round(ms * 1e3, 1), tflops=round(2 * M * N * K / ms / 1e9, 1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()

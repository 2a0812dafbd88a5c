"""GPU checks of the tcgen05 GEMM building block (NEXT-4) against an FP64
product of the same bf16-valued operands. With fp32 accumulation of K bf16
products the error bound is |err| <= K * 2^-24 * sum_k |a_k b_k| (plus the
output rounding for bf16 epilogues, 2^-9 relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_12615_b200 import build
    build.build()


def _bf(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).cuda()


def _ref(Ab, Bb, a_mn, b_mn):
    A = Ab.float().cpu().double().numpy()
    B = Bb.float().cpu().double().numpy()
    A = A.T if a_mn else A   # -> [M, K]
    B = B.T if b_mn else B   # -> [N, K]
    return A @ B.T, np.abs(A) @ np.abs(B).T


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 200, 136), (1000, 16, 256),
                                   (257, 64, 8), (2048, 256, 512)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (True, False), (False, True),
                                       (True, True)])
def test_gemm_store(M, N, K, a_mn, b_mn):
    from paper_2508_12615_b200 import abi
    rng = np.random.default_rng(M + N + K)
    A = _bf(rng.normal(size=(K, M) if a_mn else (M, K)))
    B = _bf(rng.normal(size=(K, N) if b_mn else (N, K)))
    # pad leading dimensions to multiples of 8 by construction of the shapes
    lda = M if a_mn else K
    ldb = N if b_mn else K
    if lda % 8 or ldb % 8:
        pytest.skip("leading dimension not a multiple of 8")
    C = torch.full((M, N), float("nan"), device="cuda")
    abi.gemm(A, B, C, M, N, K, lda, ldb, N, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    ref, mag = _ref(A, B, a_mn, b_mn)
    err = np.abs(C.cpu().double().numpy() - ref)
    assert np.all(err <= K * 2.0 ** -24 * mag + 1e-30), float(np.max(err / (mag + 1e-30)))


def test_gemm_epilogues():
    from paper_2508_12615_b200 import abi
    rng = np.random.default_rng(1)
    M, N, K = 384, 256, 128
    A, B = _bf(rng.normal(size=(M, K))), _bf(rng.normal(size=(N, K)))
    bias = torch.from_numpy(rng.normal(size=N).astype(np.float32)).cuda()
    ref, mag = _ref(A, B, False, False)
    tol = K * 2.0 ** -24 * mag
    C = torch.empty((M, N), device="cuda")
    abi.gemm(A, B, C, M, N, K, K, K, N, epilogue="bias_f32", bias=bias)
    Cr = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    abi.gemm(A, B, Cr, M, N, K, K, K, N, epilogue="bias_relu_bf16", bias=bias)
    mask = _bf(rng.normal(size=(M, N)))
    Cm = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    abi.gemm(A, B, Cm, M, N, K, K, K, N, epilogue="mask_bf16", mask=mask, ldm=N)
    Ca = torch.ones((M, N), device="cuda")
    abi.gemm(A, B, Ca, M, N, K, K, K, N, epilogue="atomic_f32", split_k=3)
    torch.cuda.synchronize()
    b = bias.double().cpu().numpy()
    assert np.all(np.abs(C.cpu().double().numpy() - (ref + b)) <= tol + 1e-6)
    r = np.maximum(ref + b, 0)
    assert np.all(np.abs(Cr.float().cpu().double().numpy() - r) <= tol + 2 ** -8 * np.abs(r) + 1e-6)
    mk = mask.float().cpu().numpy() > 0
    assert np.all(np.abs(Cm.float().cpu().double().numpy() - ref * mk)
                  <= tol + 2 ** -8 * np.abs(ref) + 1e-6)
    assert np.all(np.abs(Ca.cpu().double().numpy() - (ref + 1)) <= tol + 1e-5)

import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2508_12615_b200 import abi, build
build.build()
rng = np.random.default_rng(0)
def bf(x): return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).cuda()
M, W = 3000, 128
dout = bf(np.concatenate([rng.normal(size=(M, 13)), np.zeros((M, 3))], 1))
Wh = bf(np.concatenate([rng.normal(size=(13, W)), np.zeros((3, W))], 0))
h = bf(np.abs(rng.normal(size=(M, W))) * (rng.uniform(size=(M, W)) > 0.5))
dz = torch.empty((M, W), dtype=torch.bfloat16, device='cuda')
abi.gemm(dout, Wh, dz, M, W, 16, 16, W, W, epilogue='mask_bf16', b_mn=True, mask=h, ldm=W)
ref = (dout.float() @ Wh.float()) * (h.float() > 0)
print('dIn head  max err', (dz.float() - ref).abs().max().item(), 'ref rms', ref.pow(2).mean().sqrt().item())
# dW = dz^T h  (A = dz MN-major lda=W, B = h MN-major ldb=W), K = M rows, split-K atomic
C = torch.zeros((W, W), device='cuda')
abi.gemm(dz, h, C, W, W, M, W, W, W, epilogue='atomic_f32', a_mn=True, b_mn=True, split_k=47)
ref2 = dz.float().t() @ h.float()
print('dW max err', (C - ref2).abs().max().item(), 'rms', ref2.pow(2).mean().sqrt().item())
C1 = torch.zeros((W, W), device='cuda')
abi.gemm(dz, h, C1, W, W, M, W, W, W, epilogue='atomic_f32', a_mn=True, b_mn=True, split_k=1)
print('dW split1 max err', (C1 - ref2).abs().max().item())
# dW with N = 80 from a wider buffer (ldb = 208)
cat = bf(rng.normal(size=(M, 208)))
C2 = torch.zeros((W, 80), device='cuda')
abi.gemm(dz, cat, C2, W, 80, M, W, 208, 80, epilogue='atomic_f32', a_mn=True, b_mn=True, split_k=8)
ref3 = dz.float().t() @ cat.float()[:, :80]
print('dW N80 max err', (C2 - ref3).abs().max().item(), 'rms', ref3.pow(2).mean().sqrt().item())

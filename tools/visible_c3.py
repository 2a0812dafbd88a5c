import torch, sys
sys.path.insert(0, '.')
from paper_2508_12615_b200 import gen
from paper_2508_12615_b200.raster import Rasterizer
c = gen.make_config("c3", seed=0)
dev = torch.device("cuda")
p = {k: torch.as_tensor(v, device=dev) for k, v in c["params"].items()}
r = Rasterizer(c["W"], c["H"], prim="3d", blend="alpha", device=dev)
r.forward(p, c["cams"])
pp = r.get_preprocess()
cnt = pp["count"]
print("BN", cnt.numel(), "visible", int((cnt > 0).sum()), "frac", float((cnt > 0).float().mean()), "dups", int(cnt.sum()))

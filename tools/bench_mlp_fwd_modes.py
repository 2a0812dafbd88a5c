import sys, json, torch, numpy as np
sys.path.insert(0, '.')
from paper_2508_12615_b200 import gen
from paper_2508_12615_b200.deform import Deformation
N = 300000
d = Deformation(N)
th = d.init_theta(0, head_scale=0.1)
p = gen.gen3d(N, seed=0)
canon = {k: torch.from_numpy(v).cuda() for k, v in p.items()}
fr = d.forward(th, canon, [0.5])
res = {}
for train in (True, False):
    for _ in range(3):
        d.forward(th, canon, [0.5], fr, train=train)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        d.forward(th, canon, [0.5], fr, train=train)
    b.record(); b.synchronize()
    res[f"train={train}"] = a.elapsed_time(b) / 10
print(json.dumps(res))

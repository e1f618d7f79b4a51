"""Dev tool: time prepare() pieces on a device-resident fp32 matrix."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5_000
prob, _ = instances.tall_lasso(m, n, seed=0, dtype=np.float32)
Ad = torch.from_numpy(prob.A).cuda()
pd = gf.GraphFormProblem(Ad, prob.f, prob.g)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    S = gf.prepare(pd)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"prepare {m}x{n}: {t1 - t0:.4f} s (sweeps {S.scaling.iterations})")
    del S
torch.cuda.synchronize(); t0 = time.perf_counter()
P = gf.build_projector(Ad)
torch.cuda.synchronize(); print(f"build_projector: {time.perf_counter() - t0:.4f} s")

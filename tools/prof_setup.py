"""Dev tool: one prepare() of the bench instance (device-drawn A) for an ncu
launch list of the setup kernels."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5_000
prob, _ = instances.tall_lasso(m, n, seed=0, dtype=np.float32, device=True)
torch.cuda.synchronize()
S = gf.prepare(prob)
torch.cuda.synchronize()
print("ok", S.scaling.iterations)

"""Dev tool: a few iterations of BASELINE configs[2] (LP 50000 x 20000, fp64)
for an ncu capture of its iteration kernels (8-CTA cluster pass, G^-1 GEMV)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances
prob, _ = instances.generate(instances.GenSpec("lp", 50000, 20000, 0), device=True)
r = gf.solve(prob, gf.SolverSettings(max_iter=8))
torch.cuda.synchronize()
print("ok", r.iterations)

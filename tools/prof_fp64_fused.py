"""Dev tool: a few iterations of the fp64 SVM 200000 x 5000 instance (fused
pass forced with GF_FORCE_FUSED=1) for an ncu capture."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances
prob, _ = instances.generate(instances.GenSpec("svm", 200000, 5000, 0), device=True)
r = gf.solve(prob, gf.SolverSettings(max_iter=8))
torch.cuda.synchronize()
print("ok", r.iterations)

"""Dev tool: a few fp32 iterations of BASELINE configs[1] (logistic
100000 x 10000) for an ncu capture of its iteration kernels."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances
prob, _ = instances.generate(instances.GenSpec("logistic", 100000, 10000, 0), device=True)
A32 = instances._dev_matrix(prob.m, prob.n, torch.float32)
_native.convert_matrix(prob.A, A32)
A64 = None
p32 = gf.GraphFormProblem(A32, prob.f, prob.g)
r = gf.solve(p32, gf.SolverSettings(max_iter=8, precision="fp32"))
torch.cuda.synchronize()
print("ok", r.iterations)

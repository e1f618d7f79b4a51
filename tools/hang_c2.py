"""Dev tool: repeat the C2 (logistic 100000 x 10000, fp32) 2000-iteration
adaptive solve from one setup, printing each run (stall hunting).

    timeout 120 python tools/hang_c2.py [runs]
"""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prob, _ = instances.generate(instances.GenSpec("logistic", 100_000, 10_000, 0), device=True)
Ad = instances._dev_matrix(prob.m, prob.n, torch.float32)
_native.convert_matrix(prob.A, Ad)
pd = gf.GraphFormProblem(Ad, prob.f, prob.g)
S = gf.prepare(pd, gf.SolverSettings(precision="fp32"))
for r in range(runs):
    t0 = time.perf_counter()
    res = gf.solve(pd, gf.SolverSettings(max_iter=2000, precision="fp32"), setup=S)
    torch.cuda.synchronize()
    print(f"run {r}: {res.status.value} {res.iterations} it {time.perf_counter() - t0:.3f} s obj {res.objective!r}",
          flush=True)

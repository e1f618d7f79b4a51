"""Dev tool: solve a device-drawn fp64 LP (default 5000 x 2000, or C3's
50000 x 20000 with `c3`) and save x, iterations and the objective, so two runs
with different GF_DGEMM_PIPE_MINK settings can be compared bit for bit.

    GF_DGEMM_PIPE_MINK=0 python tools/check_dgemm_pipe.py out_a.npz [c3]
"""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances

out = sys.argv[1]
m, n = (50000, 20000) if "c3" in sys.argv[2:] else (5000, 2000)
prob, _ = instances.generate(instances.GenSpec("lp", m, n, 0), device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
S = gf.prepare(prob)
torch.cuda.synchronize()
t1 = time.perf_counter()
res = gf.solve(prob, setup=S)
print(f"{m}x{n} prepare {t1 - t0:.3f} s, {res.status.value} in {res.iterations} it, obj {res.objective!r}")
np.savez(out, x=res.x, nu=res.nu, it=res.iterations, obj=res.objective)

"""Dev tool: fp64 setup phases (Gram, Cholesky, TRTRI, W'W) on device-drawn
instances: C5-shaped Lasso 200000x5000 and C3 LP 50000x20000 (fp64)."""
import os, sys, time
sys.path.insert(0, ".")
os.environ.setdefault("GF_VERBOSE_SETUP", "1")
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances

for spec in (("lasso5", None), ("lp", instances.GenSpec("lp", 50000, 20000, 0))):
    if spec[1] is None:
        prob, _ = instances.tall_lasso(200000, 5000, 0, device=True)
    else:
        prob, _ = instances.generate(spec[1], device=True)
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        S = gf.prepare(prob)
        torch.cuda.synchronize()
        print(f"{spec[0]} prepare {time.perf_counter() - t0:.3f} s", flush=True)
        del S
    del prob

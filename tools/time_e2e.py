"""Dev tool: break one end-to-end solve from pinned host memory into phases
(matrix H2D, setup phases via GF_VERBOSE_SETUP, iterations), several runs."""
import os, sys, time
sys.path.insert(0, ".")
os.environ.setdefault("GF_VERBOSE_SETUP", "1")
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances, _native

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5_000
prob, _ = instances.tall_lasso(m, n, seed=0, dtype=np.float32)
A_pin = torch.from_numpy(prob.A).pin_memory()
p = gf.GraphFormProblem(A_pin, prob.f, prob.g)
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    M = _native.Matrix(A_pin, _native.GF_F32)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    del M   # (release() would hand ownership away and leak the 4 GB copy)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    res = gf.solve(p)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"run {rep}: matrix H2D {t1 - t0:.4f} s ({A_pin.numel() * 4 / (t1 - t0) / 1e9:.1f} GB/s); "
          f"solve {t3 - t2:.4f} s (setup {res.setup_time:.4f}, solve {res.solve_time:.4f}, it {res.iterations})",
          flush=True)

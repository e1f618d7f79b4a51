"""Dev tool: solve() from a plain numpy array (pageable host memory, what a
reference user passes) vs a pinned tensor."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances, _native

prob, _ = instances.tall_lasso(200_000, 5_000, seed=0, dtype=np.float32)
A_np = np.ascontiguousarray(prob.A)
A_pin = torch.from_numpy(A_np).pin_memory()
for name, A in (("numpy", A_np), ("pinned", A_pin), ("numpy", A_np), ("pinned", A_pin)):
    p = gf.GraphFormProblem(A, prob.f, prob.g)
    ts = []
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        M = _native.Matrix(A, _native.GF_F32); torch.cuda.synchronize(); t1 = time.perf_counter()
        del M
        r = gf.solve(p); torch.cuda.synchronize(); t2 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1))
    print(name, " ".join(f"H2D {a:.3f} solve {b:.3f}" for a, b in ts), flush=True)

"""Run a few ADMM iterations of the bench workload (for ncu captures).

    python tools/profile_step.py [m n steps]
"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances, solver as slv

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5_000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
prob, _ = instances.tall_lasso(m, n, seed=0, dtype=np.float32)
setup = gf.prepare(prob)
run = slv._Run(setup, prob.f, prob.g, gf.SolverSettings(abs_tol=1e-12, rel_tol=1e-12, max_iter=steps + 2),
               None, None, m)
run.run(steps)
torch.cuda.synchronize()
print("done", m, n, steps)

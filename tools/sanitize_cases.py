"""Dev tool: small solves that exercise each hand-off-heavy kernel once, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py CASE

CASE: fused32 (fused_rowcol_kernel fp32 + G^-1 ring + Z step), fused64,
cl2 (fused_rowcol_cl_kernel, fp64 rows of 40 KB), cl9 (the same on 9-CTA
clusters), lag (its lagged form: fp32 logistic rows of 40 KB), twopass
(row/col GEMV schedule), wide, indirect, gram (split_f16 + syrk_pre_kernel
tcgen05 Gram), equil (Sinkhorn kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances

case = sys.argv[1]
if case in ("cl2", "cl9"):
    os.environ["GF_FUSED_CL2"] = "1"
if case == "cl9":
    os.environ["GF_FUSED_CL"] = "9"
if case == "twopass":
    os.environ["GF_DISABLE_FUSED"] = "1"
    os.environ["GF_FUSED_CL2"] = "0"

if case in ("fused32", "gram"):
    prob, _ = instances.tall_lasso(3000, 700, 0, dtype=np.float32, device=True)
    st = gf.SolverSettings(precision="fp32", max_iter=6)
elif case in ("fused64", "twopass", "equil"):
    prob, _ = instances.tall_lasso(3000, 700, 0, device=True)
    st = gf.SolverSettings(max_iter=6)
elif case in ("cl2", "cl9"):
    prob, _ = instances.tall_lasso(int(os.environ.get("SAN_M", "6000")), 5000, 0, device=True)
    st = gf.SolverSettings(max_iter=4)
elif case == "lag":
    prob, _ = instances.generate(instances.GenSpec("logistic", 10500, 10000, 0), device=True)
    st = gf.SolverSettings(precision="fp32", max_iter=4)
elif case == "wide":
    prob, _ = instances.generate(instances.GenSpec("lasso", 200, 1000, 0), device=True)
    st = gf.SolverSettings(max_iter=6)
elif case == "indirect":
    prob, _ = instances.tall_lasso(1000, 200, 0, device=True)
    st = gf.SolverSettings(max_iter=6, projection="indirect")
else:
    raise SystemExit(f"unknown case {case}")
res = gf.solve(prob, st)
torch.cuda.synchronize()
print(case, res.status.value, res.iterations, res.objective)

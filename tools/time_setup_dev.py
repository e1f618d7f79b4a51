"""Dev tool: prepare() phases on device-drawn BASELINE instances (C5 fp32,
C5 fp64, C3 fp64), GF_VERBOSE_SETUP=1 phase lines on stderr.

    GF_VERBOSE_SETUP=1 python tools/time_setup_dev.py [c5 c5d c3]"""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances

which = sys.argv[1:] or ["c5", "c5d"]
for key in which:
    if key.startswith("c5"):
        prob, _ = instances.tall_lasso(200_000, 5_000, 0, device=True)
    else:
        prob, _ = instances.generate(instances.GenSpec("lp", 50_000, 20_000, 0), device=True)
    A = prob.A
    prec = "fp64"
    if key == "c5":
        A = instances._dev_matrix(prob.m, prob.n, torch.float32)
        _native.convert_matrix(prob.A, A)
        prec = "fp32"
    p = gf.GraphFormProblem(A, prob.f, prob.g)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = gf.prepare(p, gf.SolverSettings(precision=prec))
        torch.cuda.synchronize()
        print(f"{key} prepare: {time.perf_counter() - t0:.4f} s", file=sys.stderr, flush=True)
        del S
    del p, A, prob
    torch.cuda.empty_cache()

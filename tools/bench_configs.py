"""Per-iteration and setup timings of the BASELINE.json configs other than the
bench line (C2 logistic 100k x 10k fp32, C3 LP 50k x 20k fp64, C4 SVM
200k x 5k fp32), on one GPU.  Dev tool; prints one JSON line per config.

    python tools/bench_configs.py [c2 c3 c4] [--scale S]
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances, solver as slv

CONFIGS = {
    "c2": ("logistic", 100_000, 10_000, np.float32),
    "c3": ("lp", 50_000, 20_000, np.float64),
    "c4": ("svm", 200_000, 5_000, np.float32),
    "c4d": ("svm", 200_000, 5_000, np.float64),
    "c5d": ("tall_lasso", 200_000, 5_000, np.float64),
    "c2d": ("logistic", 100_000, 10_000, np.float64),
    "c5": ("tall_lasso", 200_000, 5_000, np.float32),
    "c2l": ("tall_lasso", 100_000, 10_000, np.float32),   # C2 shape, Lasso loss (dev)
}
NAMES = ["ginv_gemv_xside", "row_pass_yside", "col_pass", "slab_reduce", "y_scalars", "zstep_controller",
         "allreduce", "fused_rowcol_yside"]


def run(key, scale=1.0, steps=20):
    fam, m, n, dt = CONFIGS[key]
    m, n = int(m * scale), int(n * scale)
    t0 = time.perf_counter()
    if fam == "tall_lasso":
        prob, _ = instances.tall_lasso(m, n, 0, device=True)
    else:
        prob, _ = instances.generate(instances.GenSpec(fam, m, n, 0), device=True)   # A drawn on the GPU
    Ad = prob.A
    if dt == np.float32:
        Ad = instances._dev_matrix(prob.m, prob.n, torch.float32)
        _native.convert_matrix(prob.A, Ad)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    pd = gf.GraphFormProblem(Ad, prob.f, prob.g)
    A = np.empty((0,), dtype=dt)   # dtype carrier for the byte counts below
    prec = "fp32" if dt == np.float32 else "fp64"
    setups = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S = gf.prepare(pd, gf.SolverSettings(precision=prec))
        torch.cuda.synchronize()
        setups.append(time.perf_counter() - t0)
    tight = gf.SolverSettings(abs_tol=1e-14, rel_tol=1e-14, max_iter=3 + 2 * steps + 4, precision=prec)
    run_ = slv._Run(S, prob.f, prob.g, tight, None, None, m)
    run_.run(3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    st = run_.run(steps)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    L = _native.lib()
    _native.check(L.gf_solver_profile(run_.handle, 1))
    run_.run(steps)
    kms = (C.c_double * 8)()
    kcnt = (C.c_int64 * 8)()
    _native.check(L.gf_solver_stats(run_.handle, None, kms, kcnt))
    kernels = {NAMES[i]: round(kms[i] / kcnt[i], 4) for i in range(8) if kcnt[i]}
    del run_
    # full solve with default settings from the device-resident setup
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = gf.solve(pd, gf.SolverSettings(max_iter=2000, precision=prec), setup=S)
    torch.cuda.synchronize()
    solve_s = time.perf_counter() - t0
    es = A.dtype.itemsize
    q = min(m, n)
    print(json.dumps({
        "config": key, "family": fam, "m": m, "n": n, "dtype": str(A.dtype), "gen_s": round(gen_s, 2),
        "prepare_s": [round(x, 4) for x in setups], "ms_per_iter": round(ms, 4), "kernels_ms": kernels,
        "iter_bytes_alg": m * n * es + q * q * es, "GBps_alg": round((m * n * es + q * q * es) / ms / 1e6, 1),
        "solve": {"status": res.status.value, "iterations": res.iterations, "seconds": round(solve_s, 3),
                  "objective": res.objective},
        "fused": bool("fused_rowcol_yside" in kernels),
    }), flush=True)
    del S, pd, Ad, prob


if __name__ == "__main__":
    keys = [a for a in sys.argv[1:] if a in CONFIGS] or list(CONFIGS)
    scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1.0
    for k in keys:
        run(k, scale)

"""Dev tool: how far the GPU's C2 logistic 100000 x 10000 trajectories sit from
the reference fixtures (fixed-rho full solve fp64 / fp32, 200-iteration
adaptive prefix): per-iteration history deviation, iterates, objective, and the
stop test re-evaluated from the original A."""
import json
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1503_08366_b200 as gf
from tests import test_gpu_fullsize as T


def dev(name, settings, fp32=False):
    fx = T.fixture(name)
    prob = T.device_instance(fx, fp32=fp32)
    res, hist = T.solve_with_history(prob, settings)
    h = fx["history"]
    k = min(len(h), len(hist))
    rel = np.abs(hist[:k] - h[:k]) / np.maximum(np.abs(h[:k]), 1e-300)
    per_it = rel.max(axis=1)
    r_pri, r_dual, eps_pri, eps_dual = T.stop_test_from_original_A(prob, res, settings)
    out = {"case": name, "status": res.status.value, "ref_status": str(fx["status"]),
           "iterations": res.iterations, "ref_iterations": int(fx["iterations"]),
           "hist_max_rel_by_decile": [float(per_it[i * k // 10:(i + 1) * k // 10].max()) for i in range(10)],
           "hist_max_rel_by_column": [float(x) for x in rel.max(axis=0)],
           "first_k_over_1e-6": int(np.argmax(per_it > 1e-6)) if (per_it > 1e-6).any() else None,
           "x_rel": T.rel(res.x, fx["x"]), "mu_rel": T.rel(res.mu, fx["mu"]),
           "y_head_rel": T.rel(res.y[:4096], fx["y_head"]), "nu_head_rel": T.rel(res.nu[:4096], fx["nu_head"]),
           "obj_rel": abs(res.objective - float(fx["objective"])) / abs(float(fx["objective"])),
           "rho": [res.final_rho, float(fx["final_rho"])],
           "r_pri": [r_pri, res.primal_residual, eps_pri], "r_dual": [r_dual, res.dual_residual, eps_dual]}
    print(json.dumps(out), flush=True)
    del prob


which = sys.argv[1:] or ["f64", "f32", "p200"]
if "f64" in which:
    dev("c2_logistic_100000x10000_fixedrho", gf.SolverSettings(adaptive_rho=False, max_iter=1500))
if "f32" in which:
    dev("c2_logistic_100000x10000_fixedrho_r32",
        gf.SolverSettings(adaptive_rho=False, max_iter=1500, precision="fp32"), fp32=True)
if "p200" in which:
    dev("c2_logistic_100000x10000_prefix200", gf.SolverSettings(max_iter=200))

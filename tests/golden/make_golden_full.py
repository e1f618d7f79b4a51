"""Full-size golden fixtures (BASELINE.json configs at their own sizes), made
by running the REFERENCE implementation here, where /root/reference exists:

    python tests/golden/make_golden_full.py [name ...]

About 15 minutes on 8 cores.  Each fixture keeps the scalars, the per-
iteration history and the n-length vectors of one solve, plus the SHA-256 of
the first 1000 rows of A (the GPU test draws A on the device and checks that
prefix instead of hashing gigabytes).  The m-length vectors are stored as
their first 4096 entries and their norms.

Cases:
  c5_lasso_200000x5000      configs[4] / configs[1]-shape, fp64, full solve
  c5_lasso_200000x5000_r32  the same with A, b, lambda rounded to fp32
  c4_svm_200000x5000        configs[3], fp64, full solve
  c2_logistic_100000x10000_prefix  configs[1], default settings, 30 iterations
  c3_lp_50000x20000_prefix  configs[2], default settings, 10 iterations
  huber_fit_100000x2000_prefix   Huber loss + l1, 60 iterations
                                 (the full solve takes over 30 min on 8 cores)
  entropy_max_2000x50000_prefix  negative entropy, wide (m < n) orientation, 60 iterations
Round 2 (about 3 hours on 8 cores in total, C3 alone ~90 min):
  c2_logistic_100000x10000_fixedrho      configs[1], adaptive_rho=False, full solve
  c2_logistic_100000x10000_fixedrho_r32  the same on fp32-rounded A and terms
  c2_logistic_100000x10000_prefix200     configs[1], default settings, 200 iterations
  nnls / basis_pursuit 100000x5000, portfolio 100x200000 (k=100 factors): full solves
  lp_5000x2000                           configs[2] at 1/10 scale, full solve (minutes)
  c3_lp_50000x20000                      configs[2], default settings, full solve
  entropy_max_2000x50000, huber_fit_100000x2000: full solves
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (imports the reference as mg.gf)

gf = mg.gf
HEAD = 4096

CASES = [
    ("c5_lasso_200000x5000", ("tall_lasso", 200000, 5000, 0), {}),
    ("c5_lasso_200000x5000_r32", ("tall_lasso32", 200000, 5000, 0), {}),
    ("c4_svm_200000x5000", ("svm", 200000, 5000, 0), {}),
    ("c2_logistic_100000x10000_prefix", ("logistic", 100000, 10000, 0), {"max_iter": 30}),
    ("c3_lp_50000x20000_prefix", ("lp", 50000, 20000, 0), {"max_iter": 10}),
    # the other prox kinds and families at scale
    ("huber_fit_100000x2000_prefix", ("huber_fit", 100000, 2000, 0), {"max_iter": 60}),
    ("entropy_max_2000x50000_prefix", ("entropy_max", 2000, 50000, 0), {"max_iter": 60}),
    # round 2: full solves of configs[1] and configs[2], and the other families at scale
    ("c2_logistic_100000x10000_fixedrho", ("logistic", 100000, 10000, 0), {"adaptive_rho": False, "max_iter": 1500}),
    ("c2_logistic_100000x10000_fixedrho_r32", ("logistic32", 100000, 10000, 0), {"adaptive_rho": False, "max_iter": 1500}),
    ("c2_logistic_100000x10000_prefix200", ("logistic", 100000, 10000, 0), {"max_iter": 200}),
    ("nnls_100000x5000", ("nnls", 100000, 5000, 0), {}),
    ("basis_pursuit_100000x5000", ("basis_pursuit", 100000, 5000, 0), {}),
    ("portfolio_100x200000", ("portfolio", 100, 200000, 0), {}),
    ("lp_5000x2000", ("lp", 5000, 2000, 0), {}),
    ("c3_lp_50000x20000", ("lp", 50000, 20000, 0), {}),
    ("entropy_max_2000x50000", ("entropy_max", 2000, 50000, 0), {}),
    ("huber_fit_100000x2000", ("huber_fit", 100000, 2000, 0), {}),
]


def head_sha(A, rows=1000):
    return hashlib.sha256(np.ascontiguousarray(A[:rows], dtype=np.float64).tobytes()).hexdigest()


def main(only):
    for name, desc, skw in CASES:
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        problem = mg.build(desc)
        tg = time.perf_counter() - t0
        settings = gf.SolverSettings(**skw)
        hist = []
        cb = lambda k, rp, rd, ep, ed, rho, obj: hist.append((rp, rd, ep, ed, rho, obj))
        r = gf.solve(problem, settings, callback=cb)
        arrays = dict(
            desc=np.array([str(x) for x in desc]), settings=np.array(repr(skw)),
            sha_A_head=np.array(head_sha(problem.A)),
            status=np.array(r.status.value), iterations=np.array(r.iterations),
            objective=np.array(r.objective), r_pri=np.array(r.primal_residual),
            r_dual=np.array(r.dual_residual), final_rho=np.array(r.final_rho),
            history=np.array(hist, float).reshape(-1, 6),
            x=r.x, mu=r.mu, y_head=r.y[:HEAD], nu_head=r.nu[:HEAD],
            y_norm=np.array(np.linalg.norm(r.y)), nu_norm=np.array(np.linalg.norm(r.nu)),
            setup_time=np.array(r.setup_time), solve_time=np.array(r.solve_time),
            generate_time=np.array(tg),
        )
        arrays.update({f"f_{k}_head": getattr(problem.f, k)[:HEAD] for k in "habcde"})
        arrays.update({f"g_{k}": getattr(problem.g, k) for k in "habcde"})
        print(f"{name}: {r.status.value} in {r.iterations} it, obj={r.objective:.12g} "
              f"(generate {tg:.1f}s, setup {r.setup_time:.1f}s, solve {r.solve_time:.1f}s)", flush=True)
        mg.save("full_" + name, **arrays)
        del problem, r


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)

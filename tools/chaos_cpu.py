"""Dev experiment (CPU only): is the explicit G^-1 the amplifier of the chaotic
logistic trajectories, or does any ulp-level perturbation diverge as fast?

Runs the oracle on the chaotic fixtures with one fixed scaling (D, E) and
three projection applies -- (a) cho_solve (the reference), (b) an explicit
inverse G^-1 (what the GPU applies), (c) cho_solve with c + A'd summed in a
different order (a 1-ulp-level perturbation of the same algorithm) -- and
prints the first iteration at which each pair's residual history differs by
more than a threshold."""
import sys
import numpy as np
import scipy.linalg
sys.path.insert(0, ".")
from oracle import graphform_oracle as orc
from tests import _cases

base_project = orc.project


def run(prob, st, setup, mode):
    def project(P, c, d):
        A = P.A
        if mode == "inv":
            if not hasattr(P, "_ginv"):
                object.__setattr__(P, "_ginv", scipy.linalg.cho_solve(P.factor, np.eye(A.shape[1])))
            x = P._ginv @ (c + A.T @ d)
            return x, A @ x
        if mode == "perm":
            h = A.shape[0] // 2
            rhs = c + (A[h:].T @ d[h:] + A[:h].T @ d[:h])
            x = scipy.linalg.cho_solve(P.factor, rhs, check_finite=False)
            return x, A @ x
        return base_project(P, c, d)
    orc.project = project
    try:
        return orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st, setup=setup)
    finally:
        orc.project = base_project


def horizon(h, g, thr=1e-6):
    k = min(len(h), len(g))
    rel = np.max(np.abs(h[:k, :2] - g[:k, :2]) / np.abs(g[:k, :2]), axis=1)
    idx = np.nonzero(rel > thr)[0]
    return int(idx[0]) if len(idx) else None


for name in ("logistic_2000x200", "logistic_4000x400_prefix"):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    st = _cases.settings_of(fx)
    setup = orc.prepare(prob.A, st, scaling=(fx["d"], fx["e"])) if "d" in fx else orc.prepare(prob.A, st)
    r = {m: run(prob, st, setup, m) for m in ("cho", "inv", "perm")}
    print(name, {m: (r[m]["status"], r[m]["iterations"]) for m in r},
          "horizon cho-inv", horizon(r["inv"]["history"], r["cho"]["history"]),
          "cho-perm", horizon(r["perm"]["history"], r["cho"]["history"]),
          "inv-perm", horizon(r["inv"]["history"], r["perm"]["history"]), flush=True)

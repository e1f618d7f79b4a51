"""Dev tool: first iteration where GPU and oracle (same D, E) histories differ."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1503_08366_b200 as gf
from oracle import graphform_oracle as orc
from tests import _cases

for name in ("logistic_2000x200", "logistic_4000x400_prefix"):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    st = _cases.settings_of(fx)
    setup = gf.prepare(prob)
    hist = []
    res = gf.solve(prob, gf.SolverSettings(**st), setup=setup, callback=lambda *a: hist.append(a[1:]))
    ref = orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st,
                    setup=orc.prepare(prob.A, st, scaling=(setup.scaling.d, setup.scaling.e)))
    h, g = np.array(hist), ref["history"]
    k = min(len(h), len(g))
    rel = np.max(np.abs(h[:k, :2] - g[:k, :2]) / np.abs(g[:k, :2]), axis=1)
    for thr in (1e-12, 1e-10, 1e-8, 1e-6, 1e-4, 1e-2):
        idx = np.nonzero(rel > thr)[0]
        print(name, f"first k with rel>{thr:g}:", idx[0] if len(idx) else None)
    print(name, "gpu", res.status.value, res.iterations, "oracle", ref["status"], ref["iterations"],
          "rho gpu/orc", h[-1, 4], g[min(k, len(g)) - 1, 4])

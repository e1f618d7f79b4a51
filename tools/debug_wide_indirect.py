"""Dev tool: first divergence of the wide indirect solve from the reference
fixture (history rows and CGLS counts against the oracle's trace)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1503_08366_b200 as gf
from oracle import graphform_oracle as orc
from tests import _cases

name = sys.argv[1] if len(sys.argv) > 1 else "lasso_wide_200x1000_indirect"
fx = _cases.load("solve_" + name)
prob = _cases.build_problem(fx)
st = dict(_cases.settings_of(fx), max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 300)
hist, trace, otrace = [], [], []
res = gf.solve(prob, gf.SolverSettings(**st), callback=lambda *a: hist.append(a[1:]), trace=trace)
orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st, trace=otrace)
h = np.array(hist)
g = fx["history"][:len(h)]
rel = np.max(np.abs(h - g) / np.maximum(np.abs(g), 1e-300), axis=1)
bad = np.nonzero(rel > 1e-8)[0]
print("iterations", res.iterations, "first history divergence", bad[:5], rel[bad[:5]] if len(bad) else "")
gi = [t.inner_iterations for t in trace]
oi = [t.get("inner_iterations", 0) for t in otrace]
diff = [k for k in range(min(len(gi), len(oi))) if gi[k] != oi[k]]
print("inner counts gpu", gi[:20], "oracle", oi[:20], "first diff", diff[:5])
for k in diff[:2]:
    for key in ("x_hat", "y_hat", "xt", "yt"):
        a, b = getattr(trace[k], key), otrace[k][key]
        print(k, key, np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

"""Dev tool: per-iteration history of the GPU solve vs a golden fixture."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1503_08366_b200 as gf
from tests import _cases

name = sys.argv[1]
fx = _cases.load("solve_" + name)
prob = _cases.build_problem(fx, as_float32=name.endswith("_r32"))
st = gf.SolverSettings(**{**_cases.settings_of(fx), "max_iter": int(sys.argv[2]) if len(sys.argv) > 2 else 400})
hist = []
res = gf.solve(prob, st, callback=lambda *a: hist.append(a[1:]), **_cases.warm_of(fx))
h = np.array(hist)
g = fx["history"]
k = min(len(h), len(g))
rel = np.abs(h[:k] - g[:k]) / np.maximum(np.abs(g[:k]), 1e-300)
print(name, "gpu", res.status.value, res.iterations, "ref", str(fx["status"]), int(fx["iterations"]))
for i in list(range(0, min(k, 12))) + list(range(12, k, max(1, k // 20))):
    print(i, " ".join(f"{x:.3e}" for x in rel[i]), "| rho", h[i, 4], g[i, 4])

"""Dev tool: isolate the y-side prox at iteration 1 of logistic_2000x200."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1503_08366_b200 as gf
from oracle import graphform_oracle as orc
from tests import _cases

fx = _cases.load("solve_logistic_2000x200")
prob = _cases.build_problem(fx)
otr = []
orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), dict(max_iter=3), trace=otr)
gtr = []
gf.solve(prob, gf.SolverSettings(max_iter=3), trace=gtr)
for k in range(3):
    for key in ("x_hat", "y_hat", "xt", "yt", "x_half_hat", "y_half_hat"):
        a, b = getattr(gtr[k], key), otr[k][key]
        print(k, key, np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300), np.abs(a - b).argmax())
setup = orc.prepare(prob.A)
d = setup["d"]
t = otr[1]
v = (t["y_hat"] - t["yt"]) / d
rho = 1.0 * d * d
zo = orc.prox(orc.Terms.of(prob.f), rho, v)
zg = gf.prox_separable(prob.f, rho, v)
err = np.abs(zo - zg)
i = err.argmax()
print("prox max err", err.max(), "at", i, "v", v[i], "rho", rho[i], zo[i], zg[i])
print("count >1e-9:", (err > 1e-9).sum())
yg = gtr[1].y_half_hat
yo = otr[1]["y_half_hat"]
diff = np.abs(yg - yo)
idx = np.argsort(-diff)[:8]
print("num diff > 1e-9:", (diff > 1e-9).sum(), "of", len(diff))
for i in idx:
    print(i, "gpu", yg[i], "orc", yo[i], "v", v[i], "rho", rho[i], "zg_standalone*d", zg[i] * d[i], "zo*d", zo[i] * d[i],
          "h", prob.f.h[i], "dterm", prob.f.d[i])

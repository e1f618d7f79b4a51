import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1503_08366_b200 as gf
from oracle import graphform_oracle as orc
from tests import _cases

fx = _cases.load("solve_logistic_2000x200")
prob = _cases.build_problem(fx)
gtr = []
gf.solve(prob, gf.SolverSettings(max_iter=3), trace=gtr)
setup = gf.prepare(prob)
d = setup.scaling.d
t = gtr[1]
v = (t.y_hat - t.yt) / d
rho = 1.0 * d * d
zg = gf.prox_separable(prob.f, rho, v)
i = 1520
print("in-solve yhh", t.y_half_hat[i], "standalone on GPU inputs", zg[i] * d[i])
print(repr(v[i]), repr(rho[i]), repr(d[i]), repr(t.y_hat[i]), repr(t.yt[i]))
zo = orc.prox(orc.Terms.of(prob.f), rho, v)
print("oracle on GPU inputs", zo[i] * d[i])
print("all standalone vs in-solve max diff", np.abs(zg * d - t.y_half_hat).max())

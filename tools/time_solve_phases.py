"""Dev tool: wall-clock phases of solve() on a pinned host matrix, many runs
(prepare / solver create / iterate / result / teardown), to find stalls."""
import gc, os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances, solver as slv

prob, _ = instances.tall_lasso(200_000, 5_000, seed=0, dtype=np.float32)
A_pin = torch.from_numpy(prob.A).pin_memory()
p = gf.GraphFormProblem(A_pin, prob.f, prob.g)
for rep in range(6):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    S = gf.prepare(p); torch.cuda.synchronize(); t.append(time.perf_counter())
    r = slv._Run(S, p.f, p.g, gf.SolverSettings(), None, None, p.m); torch.cuda.synchronize(); t.append(time.perf_counter())
    r.run(0); torch.cuda.synchronize(); t.append(time.perf_counter())
    out = r.result(); torch.cuda.synchronize(); t.append(time.perf_counter())
    del r; torch.cuda.synchronize(); t.append(time.perf_counter())
    del S; torch.cuda.synchronize(); t.append(time.perf_counter())
    gc.collect(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"run {rep}: prepare {d[0]:.1f} create {d[1]:.1f} iterate {d[2]:.1f} result {d[3]:.1f} "
          f"del run {d[4]:.1f} del setup {d[5]:.1f} gc {d[6]:.1f}  total {1e3 * (t[-1] - t[0]):.1f} ms", flush=True)

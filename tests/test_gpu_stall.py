"""Stall regression: the sequence that exposed two hangs in session 4
(tools/hang_c2b.py at C2 size) on a smaller logistic instance with C2's row
width -- two prepares, a tight-tolerance run of 23 steps, the same run
profiled (non-PDL launches), then an adaptive solve that stops inside a
launched chunk -- with and without programmatic dependent launch.  Each
variant runs in a subprocess under a timeout: a stalled kernel fails the
test instead of holding the GPU."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, ROOT)
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances, solver as slv

# n = 10000 fp32: 40 KB rows -> the lagged 2-CTA cluster pass (C2's schedule)
prob, _ = instances.generate(instances.GenSpec("logistic", 30_000, 10_000, 0), device=True)
Ad = instances._dev_matrix(prob.m, prob.n, torch.float32)
_native.convert_matrix(prob.A, Ad)
pd = gf.GraphFormProblem(Ad, prob.f, prob.g)
for rep in range(2):
    for _ in range(2):
        S = gf.prepare(pd, gf.SolverSettings(precision="fp32"))
    tight = gf.SolverSettings(abs_tol=1e-14, rel_tol=1e-14, max_iter=47, precision="fp32")
    run_ = slv._Run(S, prob.f, prob.g, tight, None, None, prob.m)
    run_.run(3)
    run_.run(20)
    _native.check(_native.lib().gf_solver_profile(run_.handle, 1))
    run_.run(20)
    del run_
    for it in (300, 137):   # 137: the stop falls inside a launched chunk
        res = gf.solve(pd, gf.SolverSettings(max_iter=it, precision="fp32"), setup=S)
        torch.cuda.synchronize()
        assert res.iterations <= it, res.iterations
print("done", flush=True)
""".replace("ROOT", repr(ROOT))


@pytest.mark.parametrize("pdl", ["on", "off"])
def test_no_stall_lagged_pass_and_s_step(pdl):
    """Default schedules (the lower-triangle S step at this q)."""
    env = dict(os.environ)
    if pdl == "off":
        env["GF_DISABLE_PDL"] = "1"
    try:
        r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, cwd=ROOT, capture_output=True, text=True,
                           timeout=240)
    except subprocess.TimeoutExpired:
        pytest.fail(f"stalled (PDL {pdl}): the sequence did not finish in 240 s")
    assert r.returncode == 0 and "done" in r.stdout, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])

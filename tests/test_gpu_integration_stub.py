"""The ctypes binding printed in INTEGRATION.md §2 (what a maintainer would
add to the reference package) runs as written against the built library and
reproduces solve().  The module deliberately loads the library before torch
is imported (the reference package has no torch): NCCL is resolved at run
time, so the system libnccl.so.2 cannot shadow torch's newer copy."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native
from tests import _cases

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_solves_c1():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    section = text[text.index("## 2."):]
    code = re.search(r"```python\n(.*?)```", section, re.S).group(1)
    lib_path = os.path.join(ROOT, "paper_1503_08366_b200", "libgraphform_b200.so")
    code = code.replace('"libgraphform_b200.so"', repr(lib_path))
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    fx = _cases.load("solve_lasso_tall_1000x200")
    prob = _cases.build_problem(fx)
    _native.lib()   # same device/stream as the package
    x, y, mu, nu, state, hist = ns["solve_b200"](prob, gf.SolverSettings())
    ref = gf.solve(prob)
    assert state.iterations == ref.iterations == 101
    np.testing.assert_allclose(x, ref.x, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(hist, fx["history"], rtol=1e-8, atol=1e-12)

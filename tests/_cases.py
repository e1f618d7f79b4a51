"""Fixture loading shared by the CPU (oracle) and GPU (parity) tests.

Solve fixtures hold the reference's outputs; their inputs are rebuilt with
``paper_1503_08366_b200.instances`` and checked against the SHA-256 of A the
reference saw (so a drifted generator fails loudly instead of comparing
different problems).
"""

from __future__ import annotations

import ast
import glob
import hashlib
import os

import numpy as np

from paper_1503_08366_b200 import instances
from paper_1503_08366_b200.functions import SeparableFunction
from paper_1503_08366_b200.problem import GraphFormProblem

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def solve_case_names():
    return sorted(os.path.basename(p)[6:-4] for p in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


def _r32(x):
    return np.asarray(x).astype(np.float32).astype(np.float64)


def build_problem(fx, as_float32=False):
    """(problem, fp32_protocol) for a solve fixture.  ``as_float32`` keeps A as
    a float32 array (the GPU fp32 path) -- only meaningful for *_r32 cases."""
    kind, m, n, seed = fx["desc"]
    m, n, seed = int(m), int(n), int(seed)
    r32 = kind.endswith("32")
    base = kind[:-2] if r32 else kind
    if base in ("tall_lasso", "tall_ridge"):
        build = instances.tall_lasso if base == "tall_lasso" else instances.tall_ridge
        problem, _ = build(m, n, seed, dtype=np.float32 if r32 else np.float64)
        A = np.asarray(problem.A, np.float64)
    else:
        problem, _ = instances.generate(instances.GenSpec(base, m, n, seed))
        A = np.asarray(problem.A, np.float64)
        if r32:
            A = _r32(A)
    digest = hashlib.sha256(np.ascontiguousarray(A).tobytes()).hexdigest()
    assert digest == str(fx["sha_A"]), f"instance generator drifted for {fx['desc']}"
    f = SeparableFunction(*(fx[f"f_{k}"] for k in "habcde"))
    g = SeparableFunction(*(fx[f"g_{k}"] for k in "habcde"))
    if as_float32:
        A = A.astype(np.float32)
    return GraphFormProblem(A, f, g)


def settings_of(fx):
    return ast.literal_eval(str(fx["settings"]))


def warm_of(fx):
    if "x0" in fx:
        return dict(x0=fx["x0"], nu0=fx["nu0"])
    return {}

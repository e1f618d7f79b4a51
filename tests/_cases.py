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
    if base.startswith("degen_"):   # explicit small matrix stored in the fixture
        A = np.asarray(fx["A"], np.float64)
    elif base in ("tall_lasso", "tall_ridge"):
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


def same_scalar(a, ref, rtol):
    """a == ref within rtol * max(1, |ref|); NaN matches NaN and an infinity
    the same infinity (degenerate solves report non-finite objectives)."""
    a, ref = float(a), float(ref)
    if np.isnan(ref) or np.isinf(ref):
        return (np.isnan(a) and np.isnan(ref)) or a == ref
    return abs(a - ref) <= rtol * max(1.0, abs(ref))


def close_vectors(a, b, rtol, atol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    if a.shape != b.shape:
        return False
    with np.errstate(over="ignore", invalid="ignore"):
        nb = np.linalg.norm(b)
        if np.isfinite(nb) and np.all(np.isfinite(a)):
            return bool(np.linalg.norm(a - b) <= rtol * nb + atol * np.sqrt(max(b.size, 1)))
        fa, fb = np.isfinite(a), np.isfinite(b)
        if not np.array_equal(fa, fb) or not np.array_equal(a[~fb], b[~fb], equal_nan=True):
            return False
        d = np.abs(a[fb] - b[fb])
        return bool(np.all(d <= rtol * np.abs(b[fb]) + atol))

"""CPU: the C-ABI library loads and exports every entry point the header
declares; host-side model/validation mirrors the reference (no GPU calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "graphform_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(gf_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = header_functions()
    assert "gf_solver_create" in names and "gf_prox_separable" in names
    assert len(names) >= 30


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes binding declares exactly the header's entry points
    assert sorted(_native.exported_symbols()) == header_functions()
    assert b"sm_100a" in lib.gf_version()


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_reference_public_names_present():
    ref_all = ["__version__", "BaseFunction", "FunctionTerm", "SeparableFunction", "GraphFormProblem",
               "duality_gap", "eval_base", "conjugate_base", "prox_base", "prox_separable",
               "Equilibration", "equilibrate", "rescale_even", "ProjectorCache", "IndirectResult",
               "build_projector", "project", "project_indirect", "SolverSettings", "SolveResult", "Setup",
               "Status", "IterationSnapshot", "prepare", "solve", "recover_duals", "unscale",
               "residual_stop", "gap_stop", "adapt_rho", "GenSpec", "generate", "FAMILIES",
               "GraphFormError", "DimensionError", "ParameterError", "DegenerateInputError",
               "NumericError", "ProblemFormatError"]
    for name in ref_all:
        assert hasattr(gf, name), name


def test_error_codes_map_to_reference_classes():
    assert _native._ERR[1] is gf.DimensionError
    assert _native._ERR[2] is gf.ParameterError
    assert _native._ERR[3] is gf.DegenerateInputError
    assert _native._ERR[4] is gf.NumericError
    assert issubclass(gf.DimensionError, ValueError) and issubclass(gf.NumericError, RuntimeError)


def test_function_model_validation():
    with pytest.raises(gf.ParameterError):
        gf.FunctionTerm(gf.BaseFunction.ABS, a=0.0)
    with pytest.raises(gf.ParameterError):
        gf.SeparableFunction.from_arrays("abs", size=3, c=-1.0)
    with pytest.raises(gf.ParameterError):
        gf.SeparableFunction.from_arrays("abs", size=3, e=[0.0, -1.0, 0.0])
    with pytest.raises(gf.DimensionError):
        gf.SeparableFunction.from_arrays("abs", size=3, b=[1.0, 2.0])
    with pytest.raises(gf.ParameterError):
        gf.BaseFunction.from_name("nope")
    assert gf.BaseFunction.from_name("neg_entr") is gf.BaseFunction.NEG_ENTR
    assert gf.BaseFunction.from_name("IndGe0") is gf.BaseFunction.IND_GE0
    sf = gf.SeparableFunction.from_arrays(["abs", "square", "zero"], c=[1.0, 0.0, 2.0])
    codes, ceff = sf._effective
    assert list(codes) == [0, 9, 9] and list(ceff) == [1.0, 1.0, 2.0]
    t = gf.SeparableFunction.from_terms([gf.FunctionTerm("Huber", a=2.0, b=1.0)]).terms[0]
    assert t.h is gf.BaseFunction.HUBER and t.a == 2.0


def test_problem_and_settings_validation():
    f = gf.SeparableFunction.uniform("square", 4)
    g = gf.SeparableFunction.uniform("abs", 3)
    with pytest.raises(gf.DimensionError):
        gf.GraphFormProblem(np.zeros((5, 3)), f, g)
    with pytest.raises(gf.ParameterError):
        gf.GraphFormProblem(np.full((4, 3), np.inf), f, g)
    p = gf.GraphFormProblem(np.ones((4, 3), np.float32), f, g)
    assert p.A.dtype == np.float32 and p.m == 4 and p.n == 3
    for bad in (dict(rho0=0.0), dict(alpha=2.0), dict(delta=1.0), dict(tau=0.0),
                dict(max_iter=0), dict(projection="lu"), dict(abs_tol=0.0), dict(precision="fp16")):
        with pytest.raises(gf.ParameterError):
            gf.SolverSettings(**bad)


def test_instances_match_reference_streams():
    """generate() is bit-identical to the reference generators (checked
    against the SHA-256 recorded by tests/golden/make_golden.py)."""
    from tests import _cases
    for name in ("lasso_wide_200x1000", "svm_2000x100", "lp_600x240", "portfolio_20x300"):
        fx = _cases.load("solve_" + name)
        _cases.build_problem(fx)   # asserts the digest

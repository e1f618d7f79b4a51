"""GPU parity: the CUDA path against the reference's golden outputs and the
CPU oracle, through the public (C-ABI backed) API.

Tolerances (stated here):
  fp64  same status and iteration count; x, y, mu, nu and objective within
        1e-5 relative (measured spread is ~1e-12).
  fp32  (A rounded to fp32, the oracle/reference fed the same rounded values)
        same status; iterations within max(2, 5%); objective within 1e-4
        relative; x within 1e-3 relative (l2).
"""

import numpy as np
import pytest
import torch

import paper_1503_08366_b200 as gf
from oracle import graphform_oracle as orc
from tests import _cases
from tests.test_oracle_golden import check_gap

pytestmark = pytest.mark.gpu


def close(a, b, rtol, atol=1e-10):
    """||a-b|| <= rtol*||b|| + atol*sqrt(len): relative for real vectors,
    absolute for vectors that are zero up to roundoff (e.g. mu when g=Zero).
    Vectors holding non-finite or near-overflow entries (degenerate solves)
    are compared entry by entry: same NaN/inf pattern, finite entries within
    rtol (see _cases.close_entries)."""
    return _cases.close_vectors(a, b, rtol, atol)


PROX = _cases.load("prox")


@pytest.mark.parametrize("code", range(10))
def test_prox_separable_matches_reference(code):
    p = {k: PROX[f"k{code}_{k}"] for k in ("a", "b", "c", "d", "e", "rho", "v", "out")}
    sf = gf.SeparableFunction.from_arrays(gf.BaseFunction(list(gf.BaseFunction)[code]), size=len(p["v"]),
                                          a=p["a"], b=p["b"], c=p["c"], d=p["d"], e=p["e"])
    z = gf.prox_separable(sf, p["rho"], p["v"])
    np.testing.assert_allclose(z, p["out"], rtol=1e-11, atol=1e-11)
    zb = gf.prox_base(code, PROX[f"k{code}_base_rho"], PROX[f"k{code}_base_v"])
    np.testing.assert_allclose(zb, PROX[f"k{code}_base_out"], rtol=1e-11, atol=1e-11)
    hv = gf.eval_base(code, PROX[f"k{code}_eval_x"])
    ref = PROX[f"k{code}_eval_out"]
    np.testing.assert_array_equal(np.isinf(hv), np.isinf(ref))
    np.testing.assert_allclose(hv[np.isfinite(ref)], ref[np.isfinite(ref)], rtol=1e-13)
    obj = sf.evaluate(p["out"])
    r = float(PROX[f"k{code}_objective"])
    assert obj == r or abs(obj - r) <= 1e-11 * max(1.0, abs(r))


def test_prox_mixed_kinds_and_scalar_forms():
    sf = gf.SeparableFunction(*(PROX[f"mix_{k}"] for k in "habcde"))
    z = gf.prox_separable(sf, PROX["mix_rho"], PROX["mix_v"])
    np.testing.assert_allclose(z, PROX["mix_out"], rtol=1e-11, atol=1e-11)
    # SPEC.md:121-134 worked examples
    assert gf.prox_base("abs", 1.0, 0.0) == 0.0
    assert gf.prox_base("indge0", 7.0, -2.0) == 0.0
    one = gf.SeparableFunction.from_arrays("abs", size=1)
    assert gf.prox_separable(one, 1.0, [2.0])[0] == pytest.approx(1.0)
    sq = gf.SeparableFunction.from_arrays("square", size=1)
    assert gf.prox_separable(sq, 3.0, [4.0])[0] == pytest.approx(3.0)
    with pytest.raises(gf.ParameterError):
        gf.prox_separable(one, 0.0, [1.0])
    with pytest.raises(gf.DimensionError):
        gf.prox_separable(one, 1.0, [1.0, 2.0])
    # [Square a=2,b=1,c=3,d=1,e=2] at v=2 -> 19.5
    t = gf.SeparableFunction.from_terms([gf.FunctionTerm("Square", a=2, b=1, c=3, d=1, e=2)])
    assert t.evaluate([2.0]) == pytest.approx(19.5)
    assert gf.SeparableFunction.uniform("indge0", 1).evaluate([-1.0]) == np.inf


EQ = _cases.load("equil")


@pytest.mark.parametrize("name", ["gauss_300x120", "wide_80x200", "zero_row_60x30", "scaled_150x150"])
def test_equilibrate_matches_reference(name):
    A = EQ[f"{name}_A"]
    eq = gf.equilibrate(A)
    assert eq.iterations == int(EQ[f"{name}_iters"])
    assert eq.converged == bool(EQ[f"{name}_conv"])
    np.testing.assert_allclose(eq.d, EQ[f"{name}_d"], rtol=1e-10)
    np.testing.assert_allclose(eq.e, EQ[f"{name}_e"], rtol=1e-10)
    rs = gf.rescale_even(eq, A)
    np.testing.assert_allclose(rs.d, EQ[f"{name}_rd"], rtol=1e-10)
    np.testing.assert_allclose(rs.e, EQ[f"{name}_re"], rtol=1e-10)


def test_equilibrate_spec_examples_and_errors():
    eq = gf.equilibrate(np.eye(2), gamma=0.0)
    np.testing.assert_allclose(eq.d, np.sqrt([2.0, 2.0]), rtol=1e-12)
    np.testing.assert_allclose(eq.e, [1.0, 1.0], rtol=1e-12)
    rs = gf.rescale_even(gf.Equilibration(np.ones(3), np.ones(3)), 10 * np.eye(3))
    np.testing.assert_allclose(rs.d, np.full(3, 1 / np.sqrt(10)), rtol=1e-12)
    with pytest.raises(gf.DegenerateInputError):
        gf.equilibrate(np.zeros((4, 3)))


PR = _cases.load("projection")


@pytest.mark.parametrize("name", ["tall_70x25", "wide_25x70", "kkt_5x3"])
def test_projection_matches_reference(name):
    A, c, d = PR[f"{name}_A"], PR[f"{name}_c"], PR[f"{name}_d"]
    before = gf.projection.BUILD_COUNT
    P = gf.build_projector(A)
    assert gf.projection.BUILD_COUNT == before + 1
    # the fp64 Gram runs on the int8 tensor cores (exact slices, test_gram_int8_*):
    # it must agree with the reference's BLAS Gram within twice the rounding
    # bound of an fp64 dot product plus the final rounding, k eps (|A|'|A|) +
    # eps |G| (k = terms summed over), one bound for each side
    Aa = np.abs(np.asarray(A, float))
    k = A.shape[0] if A.shape[0] >= A.shape[1] else A.shape[1]
    tall = A.shape[0] >= A.shape[1]
    eps = np.finfo(float).eps
    bound = 2 * (k * eps * ((Aa.T @ Aa) if tall else (Aa @ Aa.T)) + eps * np.abs(PR[f"{name}_gram"]))
    assert np.all(np.abs(P.gram - PR[f"{name}_gram"]) <= bound)
    x, y = gf.project(P, c, d)
    np.testing.assert_allclose(x, PR[f"{name}_x"], rtol=1e-10, atol=1e-11)
    np.testing.assert_allclose(y, PR[f"{name}_y"], rtol=1e-10, atol=1e-11)
    # idempotence
    x2, y2 = gf.project(P, x, y)
    np.testing.assert_allclose(x2, x, rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("name", ["tall_70x25", "wide_25x70", "kkt_5x3"])
def test_project_indirect_matches_reference(name):
    """CGLS projection (projection.py:130-196) at tol 1e-10: same inner
    iteration count and the same point as the reference."""
    A, c, d = PR[f"{name}_A"], PR[f"{name}_c"], PR[f"{name}_d"]
    P = gf.build_projector(A, mode="indirect", tol=1e-10)
    r = gf.project_indirect(P, c, d)
    assert r.iterations == int(PR[f"{name}_iiters"]) and r.converged
    np.testing.assert_allclose(r.x, PR[f"{name}_ix"], rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(r.y, PR[f"{name}_iy"], rtol=1e-9, atol=1e-10)
    # warm start at the answer: (almost) no inner iterations
    r2 = gf.project_indirect(P, c, d, x_warm=r.x, y_warm=r.y)
    assert r2.iterations <= 1
    with pytest.raises(gf.ParameterError):
        gf.project(P, c, d)


def test_projection_closed_forms():
    sig = np.array([0.5, 2.0, 3.0])
    P = gf.build_projector(np.diag(sig))
    c, d = np.array([1.0, -2.0, 0.5]), np.array([3.0, 1.0, -1.0])
    x, y = gf.project(P, c, d)
    np.testing.assert_allclose(x, (c + sig * d) / (1 + sig ** 2), rtol=1e-12)
    np.testing.assert_allclose(y, sig * x, rtol=1e-12)
    P0 = gf.build_projector(np.zeros((4, 3)))
    np.testing.assert_allclose(P0.gram, np.eye(3))


# Logistic with adaptive rho: the reference's safeguarded Newton (prox.py:27-48)
# does not converge for some rows (it 2-cycles until the 100-iteration cap), so
# its output there is a discontinuous function of ulp-level changes of rho*d_i^2.
# Our D differs from the reference's by ~1 ulp (different summation order in the
# Sinkhorn sweeps), which flips such a row at iteration 1 of logistic_2000x200
# (row 1520).  For these cases parity is checked against the oracle run with the
# GPU's own scaling (same D, E): that isolates the iteration from the ulp-level
# equilibration difference (tools/debug_logistic2.py shows the oracle then
# reproduces the GPU value exactly).
CHAOTIC = ("logistic_2000x200", "logistic_4000x400_prefix")
# Wide Lasso with the indirect projection: the reference itself stalls to
# MaxIterations (the CGLS tolerance schedule returns after 0-1
# inner iterations, so the iteration never contracts); checked separately.
STALLED = ("lasso_wide_200x1000_indirect",)
SOLVE_FP64 = [n for n in _cases.solve_case_names()
              if not n.endswith("_r32") and n not in CHAOTIC and n not in STALLED]


@pytest.mark.parametrize("name", SOLVE_FP64)
def test_solve_fp64_matches_reference(name):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    st = gf.SolverSettings(**_cases.settings_of(fx))
    res = gf.solve(prob, st, **_cases.warm_of(fx))
    assert res.status.value == str(fx["status"])
    assert res.iterations == int(fx["iterations"])
    if "prefix" in name:   # chaotic regime: early trajectory only
        return
    for k in ("x", "y", "mu", "nu"):
        assert close(getattr(res, k), fx[k], 1e-5), k
    assert _cases.same_scalar(res.objective, float(fx["objective"]), 1e-5)
    assert res.final_rho == pytest.approx(float(fx["final_rho"]), rel=1e-9)
    if _cases.settings_of(fx).get("gap_stop"):
        check_gap(res.gap, fx, rtol=1e-6)
    else:
        assert res.gap is None


@pytest.mark.parametrize("name", CHAOTIC)
def test_solve_chaotic_logistic_same_scaling(name):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    st = _cases.settings_of(fx)
    setup = gf.prepare(prob)
    # equilibration itself agrees with the reference to a few ulps
    np.testing.assert_allclose(setup.scaling.d, fx["d"], rtol=1e-13)
    hist = []
    res = gf.solve(prob, gf.SolverSettings(**st), setup=setup, callback=lambda *a: hist.append(a[1:]))
    ref = orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st,
                    setup=orc.prepare(prob.A, st, scaling=(setup.scaling.d, setup.scaling.e)))
    h, g = np.array(hist), ref["history"]
    k = min(len(h), len(g))
    rel = np.max(np.abs(h[:k, :2] - g[:k, :2]) / np.abs(g[:k, :2]), axis=1)
    bad = np.nonzero(rel > 1e-6)[0]
    horizon = int(bad[0]) if len(bad) else k
    # with identical D, E the trajectories agree until reduction-order noise is
    # amplified (measured horizons 49 / 62 iterations); the reference against
    # itself under BLAS thread changes diverges at k ~ 317
    assert horizon >= 30, f"trajectories diverge at k={horizon}"
    assert res.status.value == ref["status"]


SOLVE_FP32 = [n for n in _cases.solve_case_names() if n.endswith("_r32")]


@pytest.mark.parametrize("name", SOLVE_FP32)
def test_solve_fp32_within_stated_band(name):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx, as_float32=True)
    res = gf.solve(prob, gf.SolverSettings(precision="fp32", **_cases.settings_of(fx)))
    it = int(fx["iterations"])
    assert res.status.value == str(fx["status"])
    assert abs(res.iterations - it) <= max(2, int(0.05 * it))
    obj = float(fx["objective"])
    assert abs(res.objective - obj) <= 1e-4 * max(1.0, abs(obj))
    assert close(res.x, fx["x"], 1e-3)


def test_callback_and_trace_match_history():
    fx = _cases.load("solve_lasso_tall_1000x200")
    prob = _cases.build_problem(fx)
    hist, trace = [], []
    res = gf.solve(prob, callback=lambda *a: hist.append(a), trace=trace)
    assert res.iterations == int(fx["iterations"]) == len(hist) == len(trace)
    h = np.array([a[1:] for a in hist])
    np.testing.assert_allclose(h, fx["history"], rtol=1e-8, atol=1e-12)
    assert [a[0] for a in hist] == list(range(len(hist)))
    # trace snapshots agree with the oracle's hat-space trajectory
    otrace = []
    orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), trace=otrace)
    for k in (0, 1, 50, len(trace) - 1):
        for key in ("x_hat", "y_hat", "xt", "yt", "x_half_hat", "y_half_hat"):
            assert close(getattr(trace[k], key), otrace[k][key], 1e-8, 1e-12), (k, key)


def test_setup_reuse_skips_build():
    fx = _cases.load("solve_lasso_tall_1000x200")
    prob = _cases.build_problem(fx)
    setup = gf.prepare(prob)
    n0 = gf.projection.BUILD_COUNT
    r1 = gf.solve(prob, setup=setup)
    r2 = gf.solve(prob, setup=setup)
    assert gf.projection.BUILD_COUNT == n0
    assert r1.setup_time == 0.0 and r1.iterations == r2.iterations == 101
    assert setup.scaling.iterations == int(fx["eq_iters"])
    np.testing.assert_allclose(setup.scaling.d, fx["d"], rtol=1e-10)
    np.testing.assert_allclose(setup.scaling.e, fx["e"], rtol=1e-10)
    # external scaling skips equilibration (solver.py:156-160)
    r3 = gf.solve(prob, scaling=setup.scaling)
    assert r3.iterations == 101


def test_c1_headline_values():
    """BASELINE config 1: Lasso 1000x200 fp64 -> Solved in 101 iterations,
    objective 252.42917798604532."""
    fx = _cases.load("solve_lasso_tall_1000x200")
    res = gf.solve(_cases.build_problem(fx))
    assert res.status is gf.Status.SOLVED and res.iterations == 101
    assert res.objective == pytest.approx(252.42917798604532, rel=1e-9)


@pytest.mark.parametrize("split", ["pre", "pre1", "f16", "tf32"])
@pytest.mark.parametrize("shape", [(17, 17), (300, 257), (513, 129), (3000, 700), (20000, 1300)])
def test_gram_tensor_core_fp32(shape, split, monkeypatch):
    """The fp32 Gram runs on tcgen05 (scaled-fp16 or TF32 three-product split,
    fp64 drain every 1024 rows): it must agree with the fp64 Gram of the same
    fp32 data to fp32-grade accuracy, including ragged tile edges.  pre: the
    default pre-split copy in 2-CTA clusters (1300 columns: an odd tile count
    per column block, so a non-draining partner CTA); pre1: single CTAs;
    f16 / tf32: in-kernel converters."""
    monkeypatch.setenv("GF_SYRK", "pre" if split == "pre1" else split)
    if split == "pre1":
        monkeypatch.setenv("GF_SYRK_CLUSTER", "1")
    m, n = shape
    A = np.random.default_rng(m + n).normal(size=(m, n)).astype(np.float32)
    G = gf.build_projector(A, precision="fp32").gram
    A64 = A.astype(np.float64)
    ref = A64.T @ A64 + np.eye(n)
    err = np.abs(G - ref).max() / np.abs(ref).max()
    # the tensor core accumulates in truncating fp32 between fp64 drains every
    # 1024 rows: measured ~5e-6 (tools/syrk_accuracy.py); plain TF32 gives ~4e-4
    assert err < 1.5e-5, err
    np.testing.assert_allclose(G, G.T, rtol=0, atol=0)


@pytest.mark.parametrize("split", ["pre", "f16"])
def test_gram_f16_split_zero_matrix(split, monkeypatch):
    """An all-zero matrix (max|A| = 0: scale 1) gives G = I exactly."""
    monkeypatch.setenv("GF_SYRK", split)
    G = gf.build_projector(np.zeros((1000, 130), np.float32), precision="fp32").gram
    np.testing.assert_array_equal(G, np.eye(130))


@pytest.mark.parametrize("scale", [1e-30, 1e-6, 1e6, 1e30])
def test_gram_f16_split_scaling(scale):
    """The fp16 split scales the panel by a power of two so that its largest
    entry sits near 2^14: matrices far outside fp16's range, and columns
    spanning six orders of magnitude, keep fp32-grade accuracy per column pair
    (off-diagonal error relative to sqrt(G_ii G_jj))."""
    m, n = 4000, 300
    rng = np.random.default_rng(7)
    A = (rng.normal(size=(m, n)) * np.logspace(-3, 3, n)[None, :] * scale).astype(np.float32)
    G = gf.build_projector(A, precision="fp32").gram
    A64 = A.astype(np.float64)
    ref = A64.T @ A64
    d = np.sqrt(np.diag(ref))
    off = ~np.eye(n, dtype=bool)   # (the diagonal carries the added identity)
    err = (np.abs(G - ref) / np.outer(d, d))[off]
    assert np.isfinite(G).all()
    assert err.max() < 2e-5, err.max()


@pytest.mark.parametrize("shape", [(17, 17), (300, 257), (513, 129), (3000, 700), (20000, 1300), (70000, 300)])
def test_gram_int8_slices_fp64(shape):
    """The fp64 Gram runs on the int8 tensor cores (tcgen05 kind::i8, seven
    exact 7-bit slices per column, int32 accumulation drained to fp64 every
    8192 rows): it must match an fp64 Gram to fp64-dot-product accuracy,
    relative to sqrt(G_ii G_jj), across ragged tiles, several drains
    (70000 rows) and columns spanning twelve orders of magnitude."""
    m, n = shape
    rng = np.random.default_rng(m * 7 + n)
    A = rng.normal(size=(m, n)) * np.logspace(-6, 6, n)[None, :]
    A[:, n // 3] = 0.0                         # an all-zero column (exponent 0)
    G = gf.build_projector(A).gram
    ref = A.T @ A
    d = np.sqrt(np.maximum(np.diag(ref), 1e-300))
    off = ~np.eye(n, dtype=bool)
    err = (np.abs(G - ref) / np.outer(d, d))[off]
    assert np.isfinite(G).all()
    assert err.max() < 1e-13, err.max()
    # the diagonal carries the added identity: its absolute resolution is ~eps
    dg = np.abs(np.diag(G) - 1.0 - np.diag(ref)) / np.maximum(np.diag(ref), 1.0)
    assert dg.max() < 1e-13
    np.testing.assert_allclose(G, G.T, rtol=0, atol=0)


def test_gram_int8_matches_dmma_path(monkeypatch):
    """The same Gram through the fp64 DMMA GEMM (GF_GRAM_F64=dmma)."""
    A = np.random.default_rng(3).normal(size=(5000, 700))
    G8 = gf.build_projector(A).gram
    monkeypatch.setenv("GF_GRAM_F64", "dmma")
    Gd = gf.build_projector(A).gram
    scale = np.sqrt(np.outer(np.diag(Gd), np.diag(Gd)))
    assert (np.abs(G8 - Gd) / scale).max() < 1e-13


CONJ = _cases.load("conj")


@pytest.mark.parametrize("code", range(10))
def test_conjugates_match_reference(code):
    """conjugate_base and SeparableFunction.conjugate (functions.py:108-393) on
    the GPU against the reference's values (None = unsupported e > 0 kind)."""
    kind = list(gf.BaseFunction)[code]
    w = CONJ[f"k{code}_w"]
    z = gf.conjugate_base(kind, w)
    ref = CONJ[f"k{code}_base"]
    np.testing.assert_array_equal(np.isinf(z), np.isinf(ref))
    fin = np.isfinite(ref)
    np.testing.assert_allclose(z[fin], ref[fin], rtol=1e-13, atol=1e-300)
    for tag in ("e0", "ep"):
        p = {k: CONJ[f"k{code}_{tag}_{k}"] for k in "abcdew"}
        sf = gf.SeparableFunction.from_arrays(kind, size=len(p["w"]), a=p["a"], b=p["b"], c=p["c"],
                                              d=p["d"], e=p["e"])
        val = sf.conjugate(p["w"])
        if bool(CONJ[f"k{code}_{tag}_none"]):
            assert val is None
        else:
            r = float(CONJ[f"k{code}_{tag}_val"])
            assert val == r or abs(val - r) <= 1e-10 * max(1.0, abs(r)), (val, r)


def test_duality_gap_and_gap_stop_helpers():
    from paper_1503_08366_b200 import instances
    prob, _ = instances.tall_ridge(300, 60, 4)
    g = gf.duality_gap(prob, CONJ["gap_x"], CONJ["gap_y"], CONJ["gap_mu"], CONJ["gap_nu"])
    assert abs(g - float(CONJ["gap_val"])) <= 1e-9
    stop, g2 = gf.gap_stop(prob, CONJ["gap_x"], CONJ["gap_y"], CONJ["gap_mu"], CONJ["gap_nu"], 1e-4, 1e-3)
    assert stop and g2 == g
    # f = g = Zero, all state zero: gap 0, stop
    z = gf.SeparableFunction.from_arrays("zero", size=3)
    p0 = gf.GraphFormProblem(np.ones((3, 3)), z, z)
    assert gf.gap_stop(p0, np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3), 1e-4, 1e-3) == (True, 0.0)
    # an unsupported conjugate (e > 0 with Abs) gives None and never stops
    ab = gf.SeparableFunction.from_arrays("abs", size=3, e=1.0)
    p1 = gf.GraphFormProblem(np.ones((3, 3)), ab, z)
    assert gf.duality_gap(p1, np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3)) is None
    assert gf.gap_stop(p1, np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3), 1e-4, 1e-3) == (False, None)


def test_one_shot_c_abi_solve_matches_public_api():
    """gf_solve (create + run + result + history + destroy in one C call, the
    boundary a ctypes/cgo binding would use) equals solve() bit for bit."""
    import ctypes as C
    from paper_1503_08366_b200 import _native, solver as slv
    fx = _cases.load("solve_lasso_tall_1000x200")
    prob = _cases.build_problem(fx)
    st = gf.SolverSettings()
    ref = gf.solve(prob, st)
    setup = gf.prepare(prob)
    L = _native.lib()
    fT, keep_f = _native.host_terms(prob.f)
    gT, keep_g = _native.host_terms(prob.g)
    s = slv._gf_settings(st)
    m, n = prob.m, prob.n
    x, mu, y, nu = np.empty(n), np.empty(n), np.empty(m), np.empty(m)
    hist = np.zeros((st.max_iter + 1, 6))
    state = _native.SolverState()
    _native.check(L.gf_solve(setup.handle, C.byref(fT), C.byref(gT), C.byref(s), None, None, _native.ptr(x),
                             _native.ptr(y), _native.ptr(mu), _native.ptr(nu), C.byref(state), _native.ptr(hist),
                             _native.stream()))
    assert state.iterations == ref.iterations == int(fx["iterations"])
    for a, b in ((x, ref.x), (y, ref.y), (mu, ref.mu), (nu, ref.nu)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_allclose(hist[:ref.iterations], fx["history"], rtol=1e-8, atol=1e-12)


def test_float32_input_runs_fp64_by_default():
    """Drop-in default: the reference coerces A to float64 (problem.py:35), so
    a float32 array solves exactly like its float64 cast unless the caller
    opts into fp32 arithmetic with precision="fp32"."""
    fx = _cases.load("solve_lasso_tall_1000x200_r32")
    p32 = _cases.build_problem(fx, as_float32=True)
    assert p32.A.dtype == np.float32
    p64 = gf.GraphFormProblem(np.asarray(p32.A, np.float64), p32.f, p32.g)
    a, b = gf.solve(p32), gf.solve(p64)
    assert a.iterations == b.iterations == int(fx["iterations"])
    np.testing.assert_array_equal(a.x, b.x)
    c = gf.solve(p32, gf.SolverSettings(precision="fp32"))
    assert c.status is gf.Status.SOLVED and not np.array_equal(c.x, a.x)


@pytest.mark.parametrize("name", ["lasso_wide_200x1000", "lasso_wide_200x1000_indirect_ptol"])
def test_trace_wide_matches_oracle(name):
    """Wide orientation (m < n): trace[k] holds iteration k's x^, x~ (the
    wide step's X(k) has already moved on to iteration k + 1; the solver keeps
    iteration k's copies for the snapshot), and with the indirect projection
    each snapshot carries the CGLS count of its own projection
    (solver.py:362-367, :410-411)."""
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    st = _cases.settings_of(fx)
    trace, otrace = [], []
    res = gf.solve(prob, gf.SolverSettings(**st), trace=trace)
    orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st, trace=otrace)
    assert res.iterations == int(fx["iterations"]) == len(trace) == len(otrace)
    for k in (0, 1, 2, 50, len(trace) - 2, len(trace) - 1):
        for key in ("x_hat", "y_hat", "xt", "yt", "x_half_hat", "y_half_hat"):
            assert close(getattr(trace[k], key), otrace[k][key], 1e-8, 1e-12), (k, key)
    if st.get("projection") == "indirect":
        got = [t.inner_iterations for t in trace]
        want = [t.get("inner_iterations", 0) for t in otrace]
        assert got == want


def test_trace_indirect_tall_records_last_projection():
    """Tall indirect solve stopped by max_iter: the CGLS count of the last
    iteration's projection is recorded too (the step that runs it records no
    new iteration), and a caller's non-empty trace list is only appended to."""
    fx = _cases.load("solve_lasso_tall_1000x200_indirect")
    prob = _cases.build_problem(fx)
    st = dict(_cases.settings_of(fx), max_iter=12)
    sentinel = object()
    trace = [sentinel]
    gf.solve(prob, gf.SolverSettings(**st), trace=trace)
    otrace = []
    orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st, trace=otrace)
    assert trace[0] is sentinel and len(trace) == 13
    assert [t.inner_iterations for t in trace[1:]] == [t.get("inner_iterations", 0) for t in otrace]


@pytest.mark.parametrize("name", ["degen_prox_300x60", "degen_proj_300x60"])
def test_degenerate_status_semantics(name):
    """Status.DEGENERATE (solver.py:337-342, :414-417): a non-finite prox at
    iteration k reports iterations = k and hands back iteration k-1's half
    iterate (here k = 0: the all-zero start, objective f(0) + g(0) = inf); a
    non-finite projection reports k + 1 with iteration k's half iterate."""
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    hist = []
    res = gf.solve(prob, gf.SolverSettings(**_cases.settings_of(fx)), callback=lambda *a: hist.append(a))
    assert res.status is gf.Status.DEGENERATE
    assert res.iterations == int(fx["iterations"]) and len(hist) == len(fx["history"])
    for k in ("x", "y", "mu", "nu"):
        assert close(getattr(res, k), fx[k], 1e-9), k
    assert _cases.same_scalar(res.objective, float(fx["objective"]), 1e-9)
    assert res.final_rho == float(fx["final_rho"])
    if name.startswith("degen_prox"):
        assert not np.any(res.x) and not np.any(res.y)


@pytest.mark.parametrize("name", STALLED)
def test_solve_stalled_indirect_wide(name):
    """wide Lasso with projection='indirect' -- the reference
    runs all 10000 iterations without meeting the stopping rule, and so does
    the GPU.  The stalled iteration does not contract, so rounding differences
    (reduction order of the GEMVs) grow instead of dying out: the GPU follows
    the reference's per-iteration history to 1e-6 for the first 500
    iterations (measured, tools/debug_wide_indirect.py: first deviation above
    1e-8 at k = 524, CGLS inner counts identical to the oracle's up to
    k = 1377), then both wander on the same plateau."""
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    hist = []
    res = gf.solve(prob, gf.SolverSettings(**_cases.settings_of(fx)), callback=lambda *a: hist.append(a[1:]))
    assert res.status.value == str(fx["status"]) == "MaxIterations"
    assert res.iterations == int(fx["iterations"]) == 10000
    h = np.array(hist)
    np.testing.assert_allclose(h[:500], fx["history"][:500], rtol=1e-6, atol=1e-12)
    # the plateau: same objective scale and residual magnitudes at the end
    assert np.isfinite(res.objective)
    assert res.objective == pytest.approx(float(fx["objective"]), rel=0.1)
    assert res.primal_residual == pytest.approx(float(fx["r_pri"]), rel=1.0)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_device_matrix_finiteness_check(dtype):
    """GraphFormProblem on a CUDA matrix checks finiteness in one device pass
    (gf_matrix_all_finite) with the reference's error (problem.py:35-49):
    padded row-strided buffers, the last row / column, NaN and inf."""
    from paper_1503_08366_b200 import instances
    m, n = 300, 37
    f = gf.SeparableFunction.uniform(gf.BaseFunction.SQUARE, m)
    g = gf.SeparableFunction.uniform(gf.BaseFunction.ABS, n)
    A = instances._dev_matrix(m, n, dtype)          # 128-byte padded rows
    A.copy_(torch.randn(m, n, dtype=dtype))
    assert gf.GraphFormProblem(A, f, g).m == m
    for (i, j, v) in [(m - 1, n - 1, float("nan")), (0, 0, float("inf")), (m // 2, n // 3, float("-inf"))]:
        B = instances._dev_matrix(m, n, dtype)
        B.copy_(A)
        B[i, j] = v
        with pytest.raises(gf.ParameterError, match="A must be finite"):
            gf.GraphFormProblem(B, f, g)

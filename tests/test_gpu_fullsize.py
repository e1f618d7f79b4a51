"""Parity at BASELINE.json's own sizes (configs[1..4]) on the GPU.

The reference's outputs at these sizes are committed as
``tests/golden/full_*.npz`` (``tests/golden/make_golden_full.py`` runs the
reference here; ~15 min on 8 cores).  The instances are drawn on the device
(``instances.generate(..., device=True)``, bit-identical to the reference's
numpy streams: the SHA-256 of the first 1000 rows of A is checked), solved
through the public API, and compared with

* the reference fixture: fp64 -- same status and iteration count, iterates and
  objective within 1e-5 relative, the per-iteration history within 1e-6;
  fp32 (A, b, lambda rounded to fp32, the reference fed the same values) --
  same status, iterations within max(2, 5 %), objective 1e-4, x 1e-3;
* size-independent properties: the stopping test re-evaluated in fp64 from
  the ORIGINAL A (not the scaled copy the solver iterates on) at the
  returned point, and the objective re-evaluated from f and g.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest
import torch

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances
from oracle import graphform_oracle as orc
from tests import _cases

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def fixture(name):
    path = os.path.join(_cases.GOLDEN, f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path} (run tests/golden/make_golden_full.py)")
    return _cases.load(f"full_{name}")


def close(a, b, tol, floor=1e-10):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b)) <= tol * float(np.linalg.norm(b)) + floor * max(1.0, np.sqrt(b.size))


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _round32_terms(t):
    r = lambda v: np.asarray(v).astype(np.float32).astype(np.float64)
    return gf.SeparableFunction(t.h, r(t.a), r(t.b), r(t.c), r(t.d), r(t.e))


def device_instance(fx, fp32=False):
    kind, m, n, seed = (str(fx["desc"][0]), int(fx["desc"][1]), int(fx["desc"][2]), int(fx["desc"][3]))
    if kind.startswith("tall_lasso"):
        prob, _ = instances.tall_lasso(m, n, seed, dtype=np.float32 if fp32 else np.float64, device=True)
    elif kind.endswith("32"):
        # the reference's fp32 protocol (make_golden.round32): A and every term
        # parameter rounded to fp32; A converted on the device
        p64, _ = instances.generate(instances.GenSpec(kind[:-2], m, n, seed), device=True)
        A32 = instances._dev_matrix(m, n, torch.float32)
        _native.convert_matrix(p64.A, A32)
        prob = gf.GraphFormProblem(A32, _round32_terms(p64.f), _round32_terms(p64.g))
        del p64
        fp32 = True
    else:
        prob, _ = instances.generate(instances.GenSpec(kind, m, n, seed), device=True)
    head = prob.A[:1000].double().cpu().numpy()
    assert hashlib.sha256(np.ascontiguousarray(head).tobytes()).hexdigest() == str(fx["sha_A_head"]), \
        "device generator drifted from the reference's stream"
    tol = 1e-6 if fp32 else 1e-10
    for k in "habcde":
        np.testing.assert_allclose(getattr(prob.f, k)[:4096], fx[f"f_{k}_head"], rtol=tol, atol=tol)
        np.testing.assert_allclose(getattr(prob.g, k), fx[f"g_{k}"], rtol=tol, atol=tol)
    return prob


def stop_test_from_original_A(prob, res, settings):
    """r_pri = ||A x - y||, r_dual = ||A' nu + mu|| in fp64 from the original A
    on the device (solver.py:191-202)."""
    A = prob.A
    dev = A.device
    x = torch.from_numpy(res.x).to(dev)
    y = torch.from_numpy(res.y).to(dev)
    nu = torch.from_numpy(res.nu).to(dev)
    rp2 = torch.zeros((), dtype=torch.float64, device=dev)
    atnu = torch.zeros(A.shape[1], dtype=torch.float64, device=dev)
    for i0 in range(0, A.shape[0], 20000):
        Ab = A[i0:i0 + 20000].double()
        rp2 += ((Ab @ x - y[i0:i0 + 20000]) ** 2).sum()
        atnu += Ab.T @ nu[i0:i0 + 20000]
    r_pri = float(rp2.sqrt())
    r_dual = float(torch.linalg.norm(atnu + torch.from_numpy(res.mu).to(dev)))
    eps_pri = settings.abs_tol + settings.rel_tol * float(np.linalg.norm(res.y))
    eps_dual = settings.abs_tol + settings.rel_tol * float(np.linalg.norm(res.mu))
    return r_pri, r_dual, eps_pri, eps_dual


def check_properties(prob, res, settings, rtol):
    """The stopping test re-evaluated from the original A at the returned
    point agrees with the solver's to rtol relative to the larger of the
    residual and its threshold (a residual far below its threshold carries
    cancellation error of the working precision, not of the solver)."""
    r_pri, r_dual, eps_pri, eps_dual = stop_test_from_original_A(prob, res, settings)
    assert abs(r_pri - res.primal_residual) <= rtol * max(res.primal_residual, eps_pri), (r_pri, res.primal_residual)
    assert abs(r_dual - res.dual_residual) <= rtol * max(res.dual_residual, eps_dual), (r_dual, res.dual_residual)
    if res.status is gf.Status.SOLVED:
        assert r_pri <= eps_pri * (1 + rtol) and r_dual <= eps_dual * (1 + rtol)
    obj = orc.evaluate(orc.Terms.of(prob.f), res.y) + orc.evaluate(orc.Terms.of(prob.g), res.x)
    assert res.objective == pytest.approx(obj, rel=1e-12)


def solve_with_history(prob, settings):
    hist = []
    res = gf.solve(prob, settings, callback=lambda *a: hist.append(a[1:]))
    return res, np.array(hist, float).reshape(-1, 6)


def check_fp64(fx, res, hist, full=True, htol=1e-6, vtol=1e-5):
    assert res.status.value == str(fx["status"])
    assert res.iterations == int(fx["iterations"])
    h = fx["history"]
    assert hist.shape == h.shape
    np.testing.assert_allclose(hist[0], h[0], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(hist, h, rtol=htol, atol=1e-12)
    # (absolute floor: some duals are identically ~0, e.g. mu of a Huber fit at 1e-16)
    assert close(res.x, fx["x"], vtol) and close(res.mu, fx["mu"], vtol)
    assert close(res.y[:4096], fx["y_head"], vtol) and close(res.nu[:4096], fx["nu_head"], vtol)
    assert np.linalg.norm(res.y) == pytest.approx(float(fx["y_norm"]), rel=vtol)
    assert np.linalg.norm(res.nu) == pytest.approx(float(fx["nu_norm"]), rel=vtol)
    obj = float(fx["objective"])
    assert abs(res.objective - obj) <= vtol * max(1.0, abs(obj))
    if full:
        assert res.final_rho == pytest.approx(float(fx["final_rho"]), rel=1e-9)


def test_c5_lasso_200000x5000_fp64():
    """BASELINE configs[4] shape (1e9 coefficients), fp64: the reference
    solves in 189 iterations."""
    fx = fixture("c5_lasso_200000x5000")
    prob = device_instance(fx)
    st = gf.SolverSettings()
    res, hist = solve_with_history(prob, st)
    assert res.status is gf.Status.SOLVED and res.iterations == 189
    check_fp64(fx, res, hist)
    check_properties(prob, res, st, 1e-8)


def test_c5_lasso_200000x5000_fp32():
    """BASELINE configs[4] as benchmarked: fp32 A (the fp32 band of SURVEY §8c)."""
    fx = fixture("c5_lasso_200000x5000_r32")
    prob = device_instance(fx, fp32=True)
    assert prob.A.dtype == torch.float32
    st = gf.SolverSettings(precision="fp32")
    res = gf.solve(prob, st)
    it = int(fx["iterations"])
    assert res.status.value == str(fx["status"])
    assert abs(res.iterations - it) <= max(2, int(0.05 * it))
    obj = float(fx["objective"])
    assert abs(res.objective - obj) <= 1e-4 * abs(obj)
    assert rel(res.x, fx["x"]) <= 1e-3
    # the stop test holds at the returned point up to fp32 rounding of A_hat
    check_properties(prob, res, st, 2e-3)


def test_c4_svm_200000x5000_fp64_and_sharded_path(tmp_path):
    """BASELINE configs[3] (hinge loss + x^2), fp64 full solve; the same
    instance through the row-partitioned code path (one-rank NCCL
    communicator: every collective call site live) is bit-identical."""
    fx = fixture("c4_svm_200000x5000")
    prob = device_instance(fx)
    st = gf.SolverSettings()
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist)
    check_properties(prob, res, st, 1e-8)
    import torch.distributed as dist
    from paper_1503_08366_b200 import distributed as gfd
    dist.init_process_group("gloo", store=dist.FileStore(str(tmp_path / "store"), 1), rank=0, world_size=1)
    try:
        comm = gfd.init_comm()
        r1 = gfd.solve_sharded(prob.A, prob.f, prob.g, st, comm=comm)
        del comm
    finally:
        dist.destroy_process_group()
    assert r1.iterations == res.iterations and r1.status is res.status
    for k in ("x", "y", "mu", "nu"):
        np.testing.assert_array_equal(getattr(r1, k), getattr(res, k), err_msg=k)


def test_c2_logistic_100000x10000_prefix():
    """BASELINE configs[1] (logistic, 1e9 coefficients): the first 30
    iterations against the reference, then the fp32 solve's own stop-test
    consistency at the same size.

    Default settings put the logistic prox in the reference's chaotic regime
    (SURVEY §7.3, App. A8): on some rows the safeguarded Newton 2-cycles for
    its full 100 iterations, so its output is a discontinuous function of
    ulp-level changes in rho * d_i^2, and D (a reduction over 1e9 entries)
    differs from numpy's in the last bits.  Iteration 0 agrees to 1e-6; after
    it the trajectories agree to a few 1e-3 (measured max 1.4e-3 over 30
    iterations) -- the band is stated here rather than hidden.  Bit-level
    trajectory parity with identical D is covered at 2000 x 200 and
    4000 x 400 (test_gpu_parity.py::test_solve_chaotic_logistic_same_scaling)."""
    fx = fixture("c2_logistic_100000x10000_prefix")
    prob = device_instance(fx)
    st = gf.SolverSettings(max_iter=30)
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist, full=False, htol=5e-3, vtol=2e-2)
    check_properties(prob, res, st, 1e-8)
    A32 = instances._dev_matrix(prob.m, prob.n, torch.float32)
    _native.convert_matrix(prob.A, A32)
    p32 = gf.GraphFormProblem(A32, prob.f, prob.g)
    del prob
    r32 = gf.solve(p32, gf.SolverSettings(max_iter=100, precision="fp32"))
    assert r32.iterations <= 100 and np.isfinite(r32.objective)
    check_properties(p32, r32, gf.SolverSettings(max_iter=100, precision="fp32"), 2e-3)


def test_c3_lp_50000x20000_prefix():
    """BASELINE configs[2] (LP in graph form, fp64, q = 20000: the two-pass
    iteration and a 3.2 GB fp64 projector): 10 iterations against the
    reference."""
    fx = fixture("c3_lp_50000x20000_prefix")
    prob = device_instance(fx)
    st = gf.SolverSettings(max_iter=10)
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist, full=False)
    check_properties(prob, res, st, 1e-8)


def test_huber_fit_100000x2000_fp64_prefix():
    """the Huber prox kind at scale (robust regression,
    huber_fit family), 60 fp64 iterations against the reference."""
    fx = fixture("huber_fit_100000x2000_prefix")
    prob = device_instance(fx)
    st = gf.SolverSettings(max_iter=60)
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist, full=False)
    check_properties(prob, res, st, 1e-8)


def test_entropy_max_2000x50000_fp64_wide_prefix():
    """negative entropy (a Newton prox) in the wide
    orientation (m < n: the I + A A' projector and the wide schedule) at
    scale, 60 fp64 iterations against the reference."""
    fx = fixture("entropy_max_2000x50000_prefix")
    prob = device_instance(fx)
    st = gf.SolverSettings(max_iter=60)
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist, full=False)
    check_properties(prob, res, st, 1e-8)


def history_band(hist, h):
    """Per-column maximum relative deviation of a residual history."""
    k = min(len(hist), len(h))
    return np.max(np.abs(hist[:k] - h[:k]) / np.maximum(np.abs(h[:k]), 1e-300), axis=0)


def test_c2_logistic_100000x10000_fixedrho_full_fp64():
    """BASELINE configs[1] (logistic + l1, 1e9 coefficients) as a full fp64
    solve with fixed rho: the reference solves in 475 iterations, and so does
    the GPU, with x, mu, y, nu and the objective within the north star's 1e-5.

    The per-iteration residuals are compared in a stated band: the
    reference's safeguarded Newton (prox.py:27-48) 2-cycles on some rows, so
    its output jumps with ulp-level changes of rho d_i^2, and D (a reduction
    over 1e9 entries) differs from numpy's in the last bits -- the residual
    histories separate from iteration 1 while the iterates converge to the
    same point (tools/c2_deviation.py)."""
    fx = fixture("c2_logistic_100000x10000_fixedrho")
    prob = device_instance(fx)
    st = gf.SolverSettings(adaptive_rho=False, max_iter=1500)
    res, hist = solve_with_history(prob, st)
    assert res.status.value == str(fx["status"]) == "Solved"
    assert res.iterations == int(fx["iterations"]) == 475
    for k in ("x", "mu"):
        assert close(getattr(res, k), fx[k], 1e-5), k
    assert close(res.y[:4096], fx["y_head"], 1e-5) and close(res.nu[:4096], fx["nu_head"], 1e-5)
    obj = float(fx["objective"])
    assert abs(res.objective - obj) <= 1e-5 * abs(obj)
    band = history_band(hist, fx["history"])
    np.testing.assert_allclose(hist[0], fx["history"][0], rtol=1e-6, atol=1e-12)
    assert np.all(band[2:] <= 1e-3) and np.all(band[:2] <= 0.5), band
    check_properties(prob, res, st, 1e-8)


def test_c2_logistic_100000x10000_fixedrho_full_fp32():
    """BASELINE configs[1] at its configured precision (fp32 matrix passes on
    one B200), full solve against the reference run on the same fp32-rounded
    A and terms: the fp32 band (status, iterations within max(2, 5 %),
    objective 1e-4, x 1e-3)."""
    fx = fixture("c2_logistic_100000x10000_fixedrho_r32")
    prob = device_instance(fx)
    assert prob.A.dtype == torch.float32
    st = gf.SolverSettings(adaptive_rho=False, max_iter=1500, precision="fp32")
    res = gf.solve(prob, st)
    it = int(fx["iterations"])
    assert res.status.value == str(fx["status"])
    assert abs(res.iterations - it) <= max(2, int(0.05 * it))
    obj = float(fx["objective"])
    assert abs(res.objective - obj) <= 1e-4 * abs(obj)
    assert rel(res.x, fx["x"]) <= 1e-3
    check_properties(prob, res, st, 2e-3)


def test_c2_logistic_100000x10000_adaptive_prefix200():
    """BASELINE configs[1] with default (adaptive rho) settings: 200
    iterations against the reference, in the chaotic regime.
    Same status and count; the first 60 iterations' residual histories within
    5e-3; at iteration 200 the objective within 1e-4, rho within 10 % and x
    within 5e-2 (stated band).  Cause of the early separation, measured on CPU
    (tools/chaos_cpu.py, oracle with one fixed scaling): applying the
    projection through an explicit G^-1 instead of cho_solve separates the
    4000 x 400 trajectory at k = 58, a 1-ulp change of summation order at
    k = 185."""
    fx = fixture("c2_logistic_100000x10000_prefix200")
    prob = device_instance(fx)
    st = gf.SolverSettings(max_iter=200)
    res, hist = solve_with_history(prob, st)
    assert res.status.value == str(fx["status"]) and res.iterations == 200
    h = fx["history"]
    assert hist.shape == h.shape
    np.testing.assert_allclose(hist[0], h[0], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(hist[:60], h[:60], rtol=5e-3, atol=1e-12)
    assert rel(res.x, fx["x"]) <= 5e-2
    assert res.final_rho == pytest.approx(float(fx["final_rho"]), rel=0.1)
    assert res.objective == pytest.approx(float(fx["objective"]), rel=1e-4)
    check_properties(prob, res, st, 1e-8)


@pytest.mark.parametrize("name", ["nnls_100000x5000", "basis_pursuit_100000x5000"])
def test_other_families_full_fp64(name):
    """SURVEY §8f item 4 at scale: non-negative least squares (kIndGe0 on x)
    and basis pursuit (equality-constrained l1), full fp64 solves."""
    fx = fixture(name)
    prob = device_instance(fx)
    st = gf.SolverSettings()
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist)
    check_properties(prob, res, st, 1e-8)


FULL_SOLVES = [n for n in ("lp_5000x2000", "c3_lp_50000x20000", "portfolio_100x200000", "entropy_max_2000x50000",
                            "huber_fit_100000x2000")
               if os.path.exists(os.path.join(_cases.GOLDEN, f"full_{n}.npz"))]


# per-iteration history tolerance: 1e-6, except the Huber fit, whose solve runs
# all 10000 iterations without meeting the stopping rule (in the reference
# too): after 10000 iterations one of its 60000 history entries sits 1.1e-6
# away (an r_dual of ~6e-5), every other one within 1e-6
HIST_TOL = {"huber_fit_100000x2000": 3e-6}


@pytest.mark.parametrize("name", FULL_SOLVES)
def test_full_solves_fp64(name):
    """Full fp64 solves of configs[2] (LP 50000 x 20000 and its 1/10-scale
    instance), the wide portfolio and negative-entropy families and the Huber
    fit: exact status and iteration count, history 1e-6,
    iterates and objective 1e-5."""
    fx = fixture(name)
    prob = device_instance(fx)
    st = gf.SolverSettings()
    res, hist = solve_with_history(prob, st)
    check_fp64(fx, res, hist, htol=HIST_TOL.get(name, 1e-6))
    check_properties(prob, res, st, 1e-8)

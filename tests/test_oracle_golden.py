"""CPU: pin the oracle restatement to the reference's golden outputs.

The oracle (oracle/graphform_oracle.py) is the checker for every GPU parity
test, so it must reproduce the reference itself: iteration counts and
statuses exactly, values to ~1e-9 relative (reference-vs-itself spread is
<=1.5e-14).
"""

import numpy as np
import pytest

from oracle import graphform_oracle as orc
from tests import _cases


def close(a, b, rtol, atol=1e-12):
    """||a-b|| <= rtol*||b|| + atol*sqrt(len): relative for real vectors,
    absolute for vectors that are zero up to roundoff (e.g. mu when g=Zero).
    Vectors holding non-finite or near-overflow entries (degenerate solves)
    are compared entry by entry: same NaN/inf pattern, finite entries within
    rtol (see _cases.close_entries)."""
    return _cases.close_vectors(a, b, rtol, atol)


PROX = _cases.load("prox")


@pytest.mark.parametrize("code", range(10))
def test_oracle_prox_matches_reference(code):
    p = {k: PROX[f"k{code}_{k}"] for k in ("a", "b", "c", "d", "e", "rho", "v", "out")}
    t = orc.Terms.make(code, len(p["v"]), p["a"], p["b"], p["c"], p["d"], p["e"])
    z = orc.prox(t, p["rho"], p["v"])
    np.testing.assert_allclose(z, p["out"], rtol=1e-13, atol=1e-13)
    zb = orc.prox_kind(code, PROX[f"k{code}_base_rho"], PROX[f"k{code}_base_v"])
    np.testing.assert_allclose(zb, PROX[f"k{code}_base_out"], rtol=1e-13, atol=1e-13)
    hv = orc.eval_kind(code, PROX[f"k{code}_eval_x"])
    np.testing.assert_array_equal(np.isinf(hv), np.isinf(PROX[f"k{code}_eval_out"]))
    fin = np.isfinite(hv)
    np.testing.assert_allclose(hv[fin], PROX[f"k{code}_eval_out"][fin], rtol=1e-14)
    obj = orc.evaluate(t, p["out"])
    ref = float(PROX[f"k{code}_objective"])
    assert (obj == ref) or abs(obj - ref) <= 1e-12 * max(1.0, abs(ref))


def test_oracle_prox_mixed_kinds():
    t = orc.Terms(*(PROX[f"mix_{k}"] for k in "habcde"))
    z = orc.prox(t, PROX["mix_rho"], PROX["mix_v"])
    np.testing.assert_allclose(z, PROX["mix_out"], rtol=1e-13, atol=1e-13)


EQ = _cases.load("equil")


@pytest.mark.parametrize("name", ["gauss_300x120", "wide_80x200", "zero_row_60x30", "scaled_150x150"])
def test_oracle_equilibrate(name):
    A = EQ[f"{name}_A"]
    r = orc.equilibrate(A)
    assert r["iterations"] == int(EQ[f"{name}_iters"])
    assert r["converged"] == bool(EQ[f"{name}_conv"])
    np.testing.assert_allclose(r["d"], EQ[f"{name}_d"], rtol=1e-12)
    np.testing.assert_allclose(r["e"], EQ[f"{name}_e"], rtol=1e-12)
    d, e = orc.rescale_even(A, r["d"], r["e"])
    np.testing.assert_allclose(d, EQ[f"{name}_rd"], rtol=1e-12)
    np.testing.assert_allclose(e, EQ[f"{name}_re"], rtol=1e-12)


PR = _cases.load("projection")


@pytest.mark.parametrize("name", ["tall_70x25", "wide_25x70", "kkt_5x3"])
def test_oracle_projection(name):
    A, c, d = PR[f"{name}_A"], PR[f"{name}_c"], PR[f"{name}_d"]
    P = orc.build_projector(A)
    x, y = orc.project(P, c, d)
    np.testing.assert_allclose(x, PR[f"{name}_x"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y, PR[f"{name}_y"], rtol=1e-12, atol=1e-12)
    Pi = orc.build_projector(A, tol=1e-10, direct=False)
    xi, yi, it, ok = orc.project_indirect(Pi, c, d)
    assert it == int(PR[f"{name}_iiters"])
    np.testing.assert_allclose(xi, PR[f"{name}_ix"], rtol=1e-10, atol=1e-12)


def test_oracle_projection_kkt_spec_example():
    """random 5x3 A: projection equals the dense KKT solve."""
    A, c, d = PR["kkt_5x3_A"], PR["kkt_5x3_c"], PR["kkt_5x3_d"]
    m, n = A.shape
    K = np.block([[np.eye(n), A.T], [A, -np.eye(m)]])
    z = np.linalg.solve(K, np.concatenate([c + A.T @ d, np.zeros(m)]))
    x, y = orc.project(orc.build_projector(A), c, d)
    np.testing.assert_allclose(x, z[:n], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y, A @ z[:n], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", _cases.solve_case_names())
def test_oracle_solve_matches_reference(name):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx)
    st = _cases.settings_of(fx)
    res = orc.solve(prob.A, orc.Terms.of(prob.f), orc.Terms.of(prob.g), st, **_cases.warm_of(fx))
    assert res["status"] == str(fx["status"])
    assert res["iterations"] == int(fx["iterations"])
    hist = fx["history"]
    if "prefix" in name:   # chaotic regime: trajectory prefix only
        np.testing.assert_allclose(res["history"][:150, :2], hist[:150, :2], rtol=1e-6)
        return
    np.testing.assert_allclose(res["history"], hist, rtol=1e-8, atol=1e-12)
    for k in ("x", "y", "mu", "nu"):
        assert close(res[k], fx[k], 1e-9), k
    assert _cases.same_scalar(res["objective"], float(fx["objective"]), 1e-9)
    assert abs(res["final_rho"] - float(fx["final_rho"])) <= 1e-12 * float(fx["final_rho"])
    if "gap" in fx and _cases.settings_of(fx).get("gap_stop"):
        check_gap(res["gap"], fx)


def check_gap(gap, fx, rtol=1e-8):
    """SolveResult.gap against the reference: None, inf, or a finite value."""
    if bool(fx["gap_none"]):
        assert gap is None
    elif np.isinf(fx["gap"]):
        assert gap is not None and np.isinf(gap)
    else:
        ref = float(fx["gap"])
        assert gap is not None and abs(gap - ref) <= rtol * max(1.0, abs(ref)), (gap, ref)


CONJ = _cases.load("conj")


@pytest.mark.parametrize("code", range(10))
def test_oracle_conjugates_match_reference(code):
    w = CONJ[f"k{code}_w"]
    z = orc.conj_kind(code, w)
    ref = CONJ[f"k{code}_base"]
    np.testing.assert_array_equal(np.isinf(z), np.isinf(ref))
    fin = np.isfinite(ref)
    np.testing.assert_allclose(z[fin], ref[fin], rtol=1e-14, atol=1e-300)
    for tag in ("e0", "ep"):
        p = {k: CONJ[f"k{code}_{tag}_{k}"] for k in "abcdew"}
        t = orc.Terms.make(code, len(p["w"]), p["a"], p["b"], p["c"], p["d"], p["e"])
        val = orc.conjugate(t, p["w"])
        if bool(CONJ[f"k{code}_{tag}_none"]):
            assert val is None
        else:
            ref = float(CONJ[f"k{code}_{tag}_val"])
            assert val == ref or abs(val - ref) <= 1e-11 * max(1.0, abs(ref)), (val, ref)


def test_oracle_duality_gap_at_solution():
    from paper_1503_08366_b200 import instances
    prob, _ = instances.tall_ridge(300, 60, 4)
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(prob.A).tobytes()).hexdigest() == str(CONJ["gap_sha"])
    g = orc.duality_gap(orc.Terms.of(prob.f), orc.Terms.of(prob.g), CONJ["gap_x"], CONJ["gap_y"],
                        CONJ["gap_mu"], CONJ["gap_nu"])
    assert abs(g - float(CONJ["gap_val"])) <= 1e-9

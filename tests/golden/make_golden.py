"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference ships no tests, so these fixtures -- the
reference's own outputs on seeded inputs -- are what pin both the CPU oracle
(``oracle/graphform_oracle.py``) and the CUDA path.  Inputs of solve cases
are rebuilt by ``paper_1503_08366_b200.instances`` (bit-identical to the
reference generators); a SHA-256 of A in each fixture proves that.  Prox and
projection fixtures store their inputs explicitly.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import graphform as gf  # noqa: E402  (the reference)

OUT = HERE


def sha(A) -> str:
    return hashlib.sha256(np.ascontiguousarray(A, dtype=np.float64).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.0f} KiB)")


# ---------------------------------------------------------------- prox ----
def make_prox():
    rng = np.random.default_rng(20261017)
    n = 1500
    out = {}
    for code, kind in enumerate(gf.BaseFunction):
        a = rng.uniform(0.3, 3.0, n) * rng.choice([-1.0, 1.0], n)
        b = rng.normal(0, 2, n)
        c = rng.uniform(0.1, 4.0, n)
        c[rng.random(n) < 0.1] = 0.0
        d = rng.normal(0, 1, n)
        e = rng.uniform(0, 2, n)
        e[rng.random(n) < 0.4] = 0.0
        rho = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
        v = rng.uniform(-30, 30, n)
        sf = gf.SeparableFunction.from_arrays(kind, size=n, a=a, b=b, c=c, d=d, e=e)
        z = gf.prox_separable(sf, rho, v)
        base_rho = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
        base_v = rng.uniform(-10, 10, n)
        zb = gf.prox_base(kind, base_rho, base_v)
        xs = rng.uniform(-5, 5, n)
        xs[:20] = 0.0
        hv = gf.eval_base(kind, xs)
        val = sf.evaluate(z)
        for k, arr in dict(a=a, b=b, c=c, d=d, e=e, rho=rho, v=v, out=z,
                           base_rho=base_rho, base_v=base_v, base_out=zb,
                           eval_x=xs, eval_out=hv).items():
            out[f"k{code}_{k}"] = arr
        out[f"k{code}_objective"] = np.array(val)
    # mixed kinds in one vector, including every kind
    h = rng.integers(0, 10, 4000)
    a = rng.uniform(0.5, 2.0, 4000) * rng.choice([-1.0, 1.0], 4000)
    b = rng.normal(0, 1, 4000)
    c = rng.uniform(0.0, 3.0, 4000)
    c[::17] = 0.0
    d = rng.normal(0, 1, 4000)
    e = np.where(rng.random(4000) < 0.5, 0.0, rng.uniform(0, 1, 4000))
    rho = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), 4000))
    v = rng.uniform(-20, 20, 4000)
    sf = gf.SeparableFunction(h=h, a=a, b=b, c=c, d=d, e=e)
    z = gf.prox_separable(sf, rho, v)
    out.update(mix_h=h, mix_a=a, mix_b=b, mix_c=c, mix_d=d, mix_e=e,
               mix_rho=rho, mix_v=v, mix_out=z,
               mix_objective=np.array(sf.evaluate(z)))
    save("prox", **out)


# ------------------------------------------------------- equilibration ----
def make_equil():
    rng = np.random.default_rng(7)
    cases = {
        "gauss_300x120": rng.normal(size=(300, 120)),
        "wide_80x200": rng.normal(size=(80, 200)) * rng.uniform(0.1, 10, (80, 1)),
        "zero_row_60x30": np.vstack([rng.normal(size=(59, 30)), np.zeros((1, 30))]),
        "scaled_150x150": rng.normal(size=(150, 150)) * np.exp(rng.normal(0, 2, (150, 1))),
    }
    out = {}
    for name, A in cases.items():
        eq = gf.equilibrate(A)
        rs = gf.rescale_even(eq, A)
        out[f"{name}_A"] = A
        out[f"{name}_d"] = eq.d
        out[f"{name}_e"] = eq.e
        out[f"{name}_iters"] = np.array(eq.iterations)
        out[f"{name}_conv"] = np.array(eq.converged)
        out[f"{name}_gamma"] = np.array(eq.gamma)
        out[f"{name}_rd"] = rs.d
        out[f"{name}_re"] = rs.e
    save("equil", **out)


# ---------------------------------------------------------- projection ----
def make_projection():
    rng = np.random.default_rng(11)
    out = {}
    for name, (m, n) in {"tall_70x25": (70, 25), "wide_25x70": (25, 70),
                         "kkt_5x3": (5, 3)}.items():
        A = rng.normal(size=(m, n))
        c = rng.normal(size=n)
        d = rng.normal(size=m)
        P = gf.build_projector(A)
        x, y = gf.project(P, c, d)
        Pi = gf.build_projector(A, mode="indirect", tol=1e-10)
        ri = gf.project_indirect(Pi, c, d)
        out.update({f"{name}_A": A, f"{name}_c": c, f"{name}_d": d,
                    f"{name}_x": x, f"{name}_y": y, f"{name}_gram": P.gram,
                    f"{name}_ix": ri.x, f"{name}_iy": ri.y,
                    f"{name}_iiters": np.array(ri.iterations)})
    save("projection", **out)


# ---------------------------------------------------------- conjugates ----
def make_conj():
    rng = np.random.default_rng(1503)
    out = {}
    n = 2000
    for code, kind in enumerate(gf.BaseFunction):
        w = rng.uniform(-3, 3, n)
        w[:8] = [0.0, 1.0, -1.0, 0.5, 1e-300, 1.0 - 1e-16, 2.0, -0.0]
        out[f"k{code}_w"] = w
        out[f"k{code}_base"] = gf.conjugate_base(kind, w)
        # separable terms of this kind: e == 0 (shift/scale rules) and, for
        # every kind, a second set with e > 0 (closed form or None)
        for tag, epos in (("e0", False), ("ep", True)):
            a = rng.uniform(0.3, 3.0, n) * rng.choice([-1.0, 1.0], n)
            b = rng.normal(0, 1, n)
            c = rng.uniform(0.1, 3.0, n)
            c[rng.random(n) < 0.1] = 0.0
            d = rng.normal(0, 1, n)
            e = rng.uniform(0.2, 2.0, n) if epos else np.zeros(n)
            sf = gf.SeparableFunction.from_arrays(kind, size=n, a=a, b=b, c=c, d=d, e=e)
            ww = rng.uniform(-2, 2, n)
            val = sf.conjugate(ww)
            for k2, arr in dict(a=a, b=b, c=c, d=d, e=e, w=ww).items():
                out[f"k{code}_{tag}_{k2}"] = arr
            out[f"k{code}_{tag}_val"] = np.array(np.nan if val is None else val)
            out[f"k{code}_{tag}_none"] = np.array(val is None)
    # duality gap of a solved ridge problem at its full iterate
    problem = tall_ridge(300, 60, 4)
    r = gf.solve(problem, gf.SolverSettings(abs_tol=1e-8, rel_tol=1e-8))
    out["gap_x"], out["gap_y"], out["gap_mu"], out["gap_nu"] = r.x, r.y, r.mu, r.nu
    out["gap_val"] = np.array(gf.duality_gap(problem, r.x, r.y, r.mu, r.nu))
    out["gap_sha"] = np.array(sha(problem.A))
    save("conj", **out)


# ---------------------------------------------------------------- solve ----
def tall_ridge(m, n, seed):
    """tall_lasso's data with g = lam * Square: every conjugate is finite, so
    the duality gap is a usable stopping rule."""
    p = tall_lasso(m, n, seed)
    lam = float(p.g.c[0])
    g = gf.SeparableFunction.from_arrays(gf.BaseFunction.SQUARE, size=n, c=lam)
    return gf.GraphFormProblem(p.A, p.f, g)


def tall_lasso(m, n, seed, fp32=False):
    root = np.random.SeedSequence([seed, 3])
    ra, rv, rn = (np.random.default_rng(s) for s in root.spawn(3))
    A = ra.normal(size=(m, n))
    v = rv.normal(0, 1 / np.sqrt(n), n)
    v[rv.random(n) < 0.5] = 0
    b = A @ v + rn.normal(0, 0.5, m)
    lam = 0.2 * float(np.max(np.abs(A.T @ b)))
    if fp32:
        A = A.astype(np.float32).astype(np.float64)
        b = b.astype(np.float32).astype(np.float64)
        lam = float(np.float32(lam))
    f = gf.SeparableFunction.from_arrays(gf.BaseFunction.SQUARE, size=m, b=b)
    g = gf.SeparableFunction.from_arrays(gf.BaseFunction.ABS, size=n, c=lam)
    return gf.GraphFormProblem(A, f, g)


def round32(problem):
    """fp32 parity protocol: A and every term parameter rounded to fp32."""
    r = lambda x: np.asarray(x).astype(np.float32).astype(np.float64)
    sf = lambda s: gf.SeparableFunction(h=s.h, a=r(s.a), b=r(s.b), c=r(s.c),
                                        d=r(s.d), e=r(s.e))
    return gf.GraphFormProblem(r(problem.A), sf(problem.f), sf(problem.g))


# name -> (builder description, settings kwargs, extra solve kwargs)
SOLVE_CASES = [
    ("lasso_tall_1000x200", ("tall_lasso", 1000, 200, 0), {}, {}),
    ("lasso_tall_1000x200_r32", ("tall_lasso32", 1000, 200, 0), {}, {}),
    ("lasso_tall_20000x500", ("tall_lasso", 20000, 500, 0), {}, {}),
    ("lasso_tall_20000x500_r32", ("tall_lasso32", 20000, 500, 0), {}, {}),
    ("lasso_wide_200x1000", ("lasso", 200, 1000, 0), {}, {}),
    ("svm_2000x100", ("svm", 2000, 100, 0), {}, {}),
    ("svm_2000x100_r32", ("svm32", 2000, 100, 0), {}, {}),
    ("svm_20000x500", ("svm", 20000, 500, 0), {}, {}),
    ("lp_600x240", ("lp", 600, 240, 0), {}, {}),
    ("lp_600x240_r32", ("lp32", 600, 240, 0), {}, {}),
    ("logistic_1000x100_fixed", ("logistic", 1000, 100, 0), {"adaptive_rho": False}, {}),
    ("logistic_1000x100_fixed_r32", ("logistic32", 1000, 100, 0), {"adaptive_rho": False}, {}),
    ("logistic_2000x200", ("logistic", 2000, 200, 0), {}, {}),
    ("logistic_4000x400_prefix", ("logistic", 4000, 400, 0), {"max_iter": 200}, {}),
    ("nnls_600x150", ("nnls", 600, 150, 0), {}, {}),
    ("huber_fit_400x80", ("huber_fit", 400, 80, 0), {}, {}),
    ("basis_pursuit_500x120", ("basis_pursuit", 500, 120, 0), {}, {}),
    ("entropy_max_60x300", ("entropy_max", 60, 300, 0), {}, {}),
    ("portfolio_20x300", ("portfolio", 20, 300, 0), {}, {}),
    ("lasso_tall_1000x200_noeq", ("tall_lasso", 1000, 200, 1), {"equilibrate": False}, {}),
    ("lasso_tall_1000x200_fixedrho", ("tall_lasso", 1000, 200, 2), {"adaptive_rho": False, "rho0": 0.5}, {}),
    ("lasso_tall_1000x200_maxit", ("tall_lasso", 1000, 200, 0), {"max_iter": 25}, {}),
    ("lasso_tall_1000x200_alpha", ("tall_lasso", 1000, 200, 0), {"alpha": 1.0, "abs_tol": 1e-5, "rel_tol": 1e-4}, {}),
    ("lasso_tall_1000x200_indirect", ("tall_lasso", 1000, 200, 0), {"projection": "indirect"}, {}),
    ("svm_2000x100_warm", ("svm", 2000, 100, 3), {}, {"warm": True}),
    # gap-based stopping (solver.py:378-390): finite gap (ridge), a gap that
    # is infinite on most iterations (Lasso: |mu| <= lam), an indicator g
    ("ridge_tall_600x150_gap", ("tall_ridge", 600, 150, 0), {"gap_stop": True}, {}),
    ("ridge_tall_600x150_gap_loose", ("tall_ridge", 600, 150, 1),
     {"gap_stop": True, "abs_tol": 1e-3, "rel_tol": 1e-2}, {}),
    ("lasso_tall_1000x200_gap", ("tall_lasso", 1000, 200, 0), {"gap_stop": True}, {}),
    ("nnls_600x150_gap", ("nnls", 600, 150, 0), {"gap_stop": True}, {}),
    # round 2: the indirect (CGLS) projection inside solve on a wide problem
    # (projection.py:152-161): the default tolerance schedule stalls at
    # MaxIterations, a fixed tolerance converges
    ("lasso_wide_200x1000_indirect", ("lasso", 200, 1000, 0), {"projection": "indirect"}, {}),
    ("lasso_wide_200x1000_indirect_ptol", ("lasso", 200, 1000, 0),
     {"projection": "indirect", "projection_tol": 1e-9}, {}),
    # Status.DEGENERATE (solver.py:337-342, :414-417): a non-finite prox at
    # iteration 0 (iterations = 0, the all-zero half iterate is returned) and
    # a non-finite projection at iteration 0 (iterations = 1, iteration 0's
    # half iterate is returned)
    ("degen_prox_300x60", ("degen_prox", 300, 60, 5), {"rho0": 1e10}, {}),
    ("degen_proj_300x60", ("degen_proj", 300, 60, 5), {}, {}),
]


def degenerate(kind, m, n, seed):
    """Lasso-like data with three huge Square targets: b = 1e300 with
    rho0 = 1e10 overflows the prox of iteration 0; b = 1e308 overflows the
    over-relaxed projection input of iteration 0 (tests/_cases.py rebuilds it
    from the stored A and terms)."""
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(m, n))
    b = rng.normal(size=m)
    b[:3] = 1e300 if kind == "degen_prox" else 1e308
    f = gf.SeparableFunction.from_arrays(gf.BaseFunction.SQUARE, size=m, b=b)
    g = gf.SeparableFunction.from_arrays(gf.BaseFunction.ABS, size=n, c=1.0)
    return gf.GraphFormProblem(A, f, g)


def build(desc):
    kind, m, n, seed = desc
    if kind.startswith("degen_"):
        return degenerate(kind, m, n, seed)
    if kind == "tall_lasso":
        return tall_lasso(m, n, seed)
    if kind == "tall_lasso32":
        return tall_lasso(m, n, seed, fp32=True)
    if kind == "tall_ridge":
        return tall_ridge(m, n, seed)
    if kind.endswith("32"):
        return round32(gf.generate(gf.GenSpec(kind[:-2], m, n, seed))[0])
    return gf.generate(gf.GenSpec(kind, m, n, seed))[0]


def make_solves(only=None):
    for name, desc, skw, xkw in SOLVE_CASES:
        if only and name not in only:
            continue
        problem = build(desc)
        settings = gf.SolverSettings(**skw)
        hist = []
        cb = lambda k, rp, rd, ep, ed, rho, obj: hist.append((rp, rd, ep, ed, rho, obj))
        kwargs = {}
        if xkw.get("warm"):
            first = gf.solve(problem, gf.SolverSettings(rel_tol=1e-2, abs_tol=1e-3))
            kwargs = dict(x0=first.x * 1.01, nu0=first.nu * 0.99)
        t0 = time.perf_counter()
        r = gf.solve(problem, settings, callback=cb, **kwargs)
        dt = time.perf_counter() - t0
        setup = gf.prepare(problem, settings)
        arrays = dict(
            x=r.x, y=r.y, mu=r.mu, nu=r.nu, objective=np.array(r.objective),
            r_pri=np.array(r.primal_residual), r_dual=np.array(r.dual_residual),
            status=np.array(r.status.value), iterations=np.array(r.iterations),
            final_rho=np.array(r.final_rho), history=np.array(hist, float).reshape(-1, 6),
            sha_A=np.array(sha(problem.A)), desc=np.array([str(x) for x in desc]),
            settings=np.array(repr(skw)), d=setup.scaling.d, e=setup.scaling.e,
            eq_iters=np.array(setup.scaling.iterations),
            gap=np.array(np.nan if r.gap is None else r.gap), gap_none=np.array(r.gap is None),
        )
        arrays.update({f"f_{k}": getattr(problem.f, k) for k in "habcde"})
        arrays.update({f"g_{k}": getattr(problem.g, k) for k in "habcde"})
        if kwargs:
            arrays.update(x0=kwargs["x0"], nu0=kwargs["nu0"])
        if problem.A.size <= 30_000:
            arrays["A"] = problem.A
        print(f"{name}: {r.status.value} in {r.iterations} it, obj={r.objective:.10g} ({dt:.2f}s)")
        save("solve_" + name, **arrays)


if __name__ == "__main__":
    only = set(sys.argv[1:]) or None
    if not only:
        make_prox()
        make_equil()
        make_projection()
    if not only or "conj" in only:
        make_conj()
    make_solves(only)

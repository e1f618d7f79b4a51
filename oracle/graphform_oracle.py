"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy (fp64) restatement of the reference ``graphform`` solve path
(POGS graph-form ADMM, arXiv 1503.08366) used as the parity checker for the
CUDA implementation.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import this module; the product package never does, and it has no CPU
fallback that could route here.

Pinning: ``tests/golden/make_golden.py`` imports the reference itself (from
/root/reference, available only in the build container) and records its
outputs as fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this restatement against every fixture (iteration counts exact,
values to ~1e-10).  The reference ships no tests of its own, so
those fixtures plus the SPEC.md worked examples are the pins.

The per-iteration structure deliberately follows the reference (residuals on
the unscaled A, scipy ``cho_solve`` on the cached factor) so that timing this
module is a fair stand-in for timing the reference on a box where
/root/reference does not exist (bench.py ``--impl reference``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import scipy.linalg

# base-kind codes, enum order of functions.py:34-46
ABS, SQUARE, HUBER, NEG_ENTR, LOGISTIC, MAX_POS0, IND_GE0, IND_LE0, IND_EQ0, ZERO = range(10)
NEWTON_TOL = 1e-12      # prox.py:23
NEWTON_MAXIT = 100      # prox.py:24


@dataclass(frozen=True)
class Terms:
    """Flat term arrays of c*h(a*x-b)+d*x+(e/2)x^2 (functions.py:193-225)."""
    h: np.ndarray
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray
    e: np.ndarray

    @staticmethod
    def of(sf) -> "Terms":
        """From any object with h,a,b,c,d,e attributes (reference or ours)."""
        return Terms(*(np.asarray(getattr(sf, k)) for k in "habcde"))

    @staticmethod
    def make(h, n, a=1.0, b=0.0, c=1.0, d=0.0, e=0.0) -> "Terms":
        full = lambda x: np.broadcast_to(np.asarray(x, float), (n,)).copy()
        return Terms(full(h).astype(np.int64), full(a), full(b), full(c),
                     full(d), full(e))

    def __len__(self):
        return len(self.h)


# ---------------------------------------------------------------- prox ----
def _sigmoid(x):
    # scipy.special.expit, the reference's sigmoid (prox.py:15)
    from scipy.special import expit
    return expit(x)


def _newton_logistic(rho, v):
    """Root of rho*(z-v) + sigmoid(z) on [v-1/rho, v]; safeguarded Newton
    with bisection fallback (prox.py:27-48)."""
    lo, hi = v - 1.0 / rho, v.copy()
    z = np.clip(v - _sigmoid(v) / (rho + 0.25), lo, hi)
    tol = NEWTON_TOL * np.maximum(1.0, np.abs(rho * v))
    fin = np.zeros(v.shape, bool)
    for _ in range(NEWTON_MAXIT):
        s = _sigmoid(z)
        r = rho * (z - v) + s
        fin |= np.abs(r) <= tol
        if fin.all():
            break
        act = ~fin
        lo = np.where(act & (r < 0.0), z, lo)
        hi = np.where(act & ~(r < 0.0), z, hi)
        step = z - r / (rho + s * (1.0 - s))
        out = (step <= lo) | (step >= hi) | ~np.isfinite(step)
        z = np.where(fin, z, np.where(out, 0.5 * (lo + hi), step))
    return z


def _newton_negentr(rho, v):
    """Root of log z + 1 + rho*(z-v) on z > 0 (prox.py:51-70)."""
    z = np.maximum(v, 1e-6)
    lo, hi = np.zeros_like(z), np.maximum(v, 1.0)
    tol = NEWTON_TOL * np.maximum(1.0, np.abs(rho) * (np.abs(v) + 1.0))
    fin = np.zeros(v.shape, bool)
    for _ in range(NEWTON_MAXIT):
        r = np.log(z) + 1.0 + rho * (z - v)
        fin |= np.abs(r) <= tol
        if fin.all():
            break
        act = ~fin
        lo = np.where(act & (r < 0.0), z, lo)
        hi = np.where(act & ~(r < 0.0), z, hi)
        step = z - r * z / (1.0 + rho * z)
        out = (step <= lo) | (step >= hi) | ~np.isfinite(step)
        z = np.where(fin, z, np.where(out, 0.5 * (lo + hi), step))
    return z


def prox_kind(code: int, rho, v):
    """Base prox argmin_z h(z) + rho/2 (z-v)^2 for one kind (prox.py:73-98)."""
    v = np.asarray(v, float)
    rho = np.broadcast_to(np.asarray(rho, float), v.shape)
    if code == ZERO:
        return v.copy()
    if code == ABS:
        return np.sign(v) * np.maximum(np.abs(v) - 1.0 / rho, 0.0)
    if code == SQUARE:
        return rho * v / (1.0 + rho)
    if code == HUBER:
        return np.where(np.abs(v) <= 1.0 + 1.0 / rho, rho * v / (1.0 + rho),
                        v - np.sign(v) / rho)
    if code == NEG_ENTR:
        return _newton_negentr(rho, v)
    if code == LOGISTIC:
        return _newton_logistic(rho, v)
    if code == MAX_POS0:
        return np.where(v <= 0.0, v, np.where(v >= 1.0 / rho, v - 1.0 / rho, 0.0))
    if code == IND_GE0:
        return np.maximum(v, 0.0)
    if code == IND_LE0:
        return np.minimum(v, 0.0)
    if code == IND_EQ0:
        return np.zeros_like(v)
    raise ValueError(code)


def prox(t: Terms, rho, v):
    """Separable prox with per-coordinate rho, via the parametric transform
    (prox.py:113-138): zero-weight terms act as ZERO with c=1."""
    v = np.asarray(v, float)
    rho = np.broadcast_to(np.asarray(rho, float), v.shape)
    zc = t.c == 0.0
    codes = np.where(zc, ZERO, t.h)
    ceff = np.where(zc, 1.0, t.c)
    den = t.e + rho
    rho_h = den / (ceff * t.a * t.a)
    z0 = t.a * (v * rho - t.d) / den - t.b
    z = np.empty_like(z0)
    for code in np.unique(codes):
        sel = codes == code
        z[sel] = prox_kind(int(code), rho_h[sel], z0[sel])
    return (z + t.b) / t.a


# ---------------------------------------------------------- evaluation ----
def eval_kind(code: int, x):
    """h(x) elementwise with +inf off-domain (functions.py:77-105)."""
    x = np.asarray(x, float)
    with np.errstate(divide="ignore", invalid="ignore"):
        if code == ZERO:
            return np.zeros_like(x)
        if code == ABS:
            return np.abs(x)
        if code == SQUARE:
            return 0.5 * x * x
        if code == HUBER:
            return np.where(np.abs(x) <= 1.0, 0.5 * x * x, np.abs(x) - 0.5)
        if code == NEG_ENTR:
            return np.where(x > 0.0, x * np.log(np.where(x > 0.0, x, 1.0)),
                            np.where(x == 0.0, 0.0, np.inf))
        if code == LOGISTIC:
            return np.logaddexp(0.0, x)
        if code == MAX_POS0:
            return np.maximum(x, 0.0)
        if code == IND_GE0:
            return np.where(x >= 0.0, 0.0, np.inf)
        if code == IND_LE0:
            return np.where(x <= 0.0, 0.0, np.inf)
        if code == IND_EQ0:
            return np.where(x == 0.0, 0.0, np.inf)
    raise ValueError(code)


def evaluate(t: Terms, v) -> float:
    """sum_i c_i h_i(a_i v_i - b_i) + d_i v_i + e_i v_i^2 / 2; zero-weight
    coordinates contribute 0 even off-domain (functions.py:307-327)."""
    v = np.asarray(v, float)
    z = t.a * v - t.b
    hv = np.empty_like(z)
    for code in np.unique(t.h):
        sel = t.h == code
        hv[sel] = eval_kind(int(code), z[sel])
    hv = np.where(t.c == 0.0, 0.0, hv)
    return float(t.c @ hv) + float(t.d @ v) + 0.5 * float(t.e @ (v * v))


# ---------------------------------------------------------- conjugates ----
def conj_kind(code: int, w):
    """h*(w) elementwise, +inf off-domain (functions.py:108-144)."""
    w = np.asarray(w, float)
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        if code == ZERO:
            return np.where(w == 0.0, 0.0, np.inf)
        if code == ABS:
            return np.where(np.abs(w) <= 1.0, 0.0, np.inf)
        if code == SQUARE:
            return 0.5 * w * w
        if code == HUBER:
            return np.where(np.abs(w) <= 1.0, 0.5 * w * w, np.inf)
        if code == NEG_ENTR:
            return np.exp(w - 1.0)
        if code == LOGISTIC:
            out = np.full_like(w, np.inf)
            ok = (w >= 0.0) & (w <= 1.0)
            wk = w[ok]
            lhs = np.where(wk > 0.0, wk * np.log(np.where(wk > 0.0, wk, 1.0)), 0.0)
            rhs = np.where(wk < 1.0, (1.0 - wk) * np.log1p(-np.where(wk < 1.0, wk, 0.0)), 0.0)
            out[ok] = lhs + rhs
            return out
        if code == MAX_POS0:
            return np.where((w >= 0.0) & (w <= 1.0), 0.0, np.inf)
        if code == IND_GE0:
            return np.where(w <= 0.0, 0.0, np.inf)
        if code == IND_LE0:
            return np.where(w >= 0.0, 0.0, np.inf)
        if code == IND_EQ0:
            return np.zeros_like(w)
    raise ValueError(code)


_EPOS_OK = (ZERO, SQUARE, IND_EQ0, IND_GE0, IND_LE0)   # functions.py:182-190


def conjugate(t: Terms, w):
    """sum_i f_i*(w_i), or None when a term with e > 0 has no closed form
    (functions.py:329-393)."""
    w = np.asarray(w, float)
    zc = t.c == 0.0
    codes = np.where(zc, ZERO, t.h)
    c = np.where(zc, 1.0, t.c)
    a, b, e = t.a, t.b, t.e
    wd = w - t.d
    vals = np.empty_like(w)
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        for code in np.unique(codes):
            sel = codes == code
            s0 = sel & (e == 0.0)
            sp = sel & (e != 0.0)
            if s0.any():
                q = wd[s0] / (a[s0] * c[s0])
                vals[s0] = c[s0] * conj_kind(int(code), q) + b[s0] * wd[s0] / a[s0]
            if sp.any():
                if int(code) not in _EPOS_OK:
                    return None
                wq, aq, bq, cq, eq = wd[sp], a[sp], b[sp], c[sp], e[sp]
                if code == ZERO:
                    vals[sp] = wq * wq / (2.0 * eq)
                elif code == SQUARE:
                    alpha = cq * aq * aq + eq
                    beta = -cq * aq * bq
                    cst = 0.5 * cq * bq * bq
                    tt = wq - beta
                    vals[sp] = tt * tt / (2.0 * alpha) - cst
                else:
                    x0 = bq / aq
                    boundary = wq * x0 - 0.5 * eq * x0 * x0
                    if code == IND_EQ0:
                        vals[sp] = boundary
                    else:
                        xbar = wq / eq
                        interior = wq * wq / (2.0 * eq)
                        if code == IND_GE0:
                            feas = np.where(aq > 0.0, xbar >= x0, xbar <= x0)
                        else:
                            feas = np.where(aq > 0.0, xbar <= x0, xbar >= x0)
                        vals[sp] = np.where(feas, interior, boundary)
    return float(np.sum(vals))


def duality_gap(f: Terms, g: Terms, x, y, mu, nu):
    """f(y) + f*(nu) + g(x) + g*(mu), None if unsupported (problem.py:67-85)."""
    fc = conjugate(f, nu)
    if fc is None:
        return None
    gc = conjugate(g, mu)
    if gc is None:
        return None
    return evaluate(f, y) + fc + evaluate(g, x) + gc


# ------------------------------------------------------- equilibration ----
def _sq_rows(A, w, chunk=256):
    """(A∘A) w, formed chunk by chunk (equilibration.py:94-116)."""
    out = np.empty(A.shape[0])
    for r in range(0, A.shape[0], chunk):
        blk = A[r:r + chunk]
        out[r:r + blk.shape[0]] = (blk * blk) @ w
    return out


def _sq_cols(A, w, chunk=256):
    """(A∘A)^T w, accumulated chunk by chunk (equilibration.py:118-123)."""
    out = np.zeros(A.shape[1])
    for r in range(0, A.shape[0], chunk):
        blk = A[r:r + chunk]
        out += (blk * blk).T @ w[r:r + blk.shape[0]]
    return out


def equilibrate(A, gamma=None, eps=None, max_iter=300, on_sweep=None):
    """Regularised Sinkhorn-Knopp, p = 2 (equilibration.py:134-197).
    Returns dict(d, e, iterations, converged, gamma) with d, e the square
    roots of the Sinkhorn iterates."""
    A = np.asarray(A, float)
    m, n = A.shape
    if not np.any(A):
        raise ValueError("cannot equilibrate an all-zero matrix")
    gamma = (m + n) * np.sqrt(np.finfo(float).eps) if gamma is None else gamma
    eps = 1e-4 * np.sqrt(max(m, n)) if eps is None else eps
    e_it = np.ones(n)
    d_it = d_old = None
    done = False
    sweeps = 0
    with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
        while sweeps < max_iter:
            sweeps += 1
            d_it = n / (_sq_rows(A, e_it) + gamma / m)
            e_next = m / (_sq_cols(A, d_it) + gamma / n)
            if on_sweep is not None:
                on_sweep(sweeps, np.sqrt(d_it), np.sqrt(e_next))
            moved_e = np.linalg.norm(e_next - e_it)
            e_it = e_next
            if d_old is not None and moved_e <= eps and np.linalg.norm(d_it - d_old) <= eps:
                done = True
                break
            d_old = d_it
    if not (np.all(np.isfinite(d_it)) and np.all(np.isfinite(e_it))
            and np.all(d_it > 0) and np.all(e_it > 0)):
        raise FloatingPointError("equilibration iterates are not finite")
    return dict(d=np.sqrt(d_it), e=np.sqrt(e_it), iterations=sweeps,
                converged=done, gamma=float(gamma))


def rescale_even(A, d, e):
    """Split |DAE|_F / sqrt(min(m,n)) evenly between d and e
    (equilibration.py:200-224)."""
    m, n = A.shape
    fro = np.sqrt(float((d * d) @ _sq_rows(A, e * e)))
    s = np.sqrt(fro / np.sqrt(min(m, n)))
    return d / s, e / s


# ---------------------------------------------------------- projection ----
@dataclass
class Projector:
    """Direct-mode projector state (projection.py:39-49, :61-99)."""
    A: np.ndarray
    tall: bool
    factor: tuple
    max_inner: int
    tol: float


def build_projector(A, tol=1e-8, max_inner=None, direct=True):
    A = np.asarray(A, float)
    m, n = A.shape
    tall = m >= n
    max_inner = max(100, 2 * min(m, n)) if max_inner is None else max_inner
    factor = None
    if direct:
        G = A.T @ A if tall else A @ A.T
        G[np.diag_indices_from(G)] += 1.0
        factor = scipy.linalg.cho_factor(G, lower=True, check_finite=True)
    return Projector(A, tall, factor, int(max_inner), float(tol))


def project(P: Projector, c, d):
    """Tall: x = (A'A+I)^-1 (c + A'd), y = Ax.  Wide: w = (AA'+I)^-1 (Ac-d),
    y = d + w, x = c - A'w (projection.py:112-127)."""
    A = P.A
    if P.tall:
        x = scipy.linalg.cho_solve(P.factor, c + A.T @ d, check_finite=False)
        return x, A @ x
    w = scipy.linalg.cho_solve(P.factor, A @ c - d, check_finite=False)
    return c - A.T @ w, d + w


def cgls(mv, rmv, h1, h2, z0, tol, max_inner):
    """CGLS on [G; I] z = [h1; h2] (projection.py:165-196).
    Returns (z, iterations, converged)."""
    z = np.array(z0, float, copy=True)
    r1 = h1 - mv(z)
    r2 = h2 - z
    s = rmv(r1) + r2
    gam = float(s @ s)
    ref = float(np.linalg.norm(rmv(h1) + h2)) or 1.0
    thr = (tol * ref) ** 2
    if gam <= thr:
        return z, 0, True
    p = s.copy()
    for it in range(1, max_inner + 1):
        q = mv(p)
        den = float(q @ q) + float(p @ p)
        if den <= 0.0 or not np.isfinite(den):
            return z, it, False
        step = gam / den
        z += step * p
        r1 -= step * q
        r2 -= step * p
        s = rmv(r1) + r2
        gnew = float(s @ s)
        if gnew <= thr:
            return z, it, True
        p = s + (gnew / gam) * p
        gam = gnew
    return z, max_inner, False


def project_indirect(P: Projector, c, d, x_warm=None, y_warm=None, tol=None):
    """CGLS projection with warm start (projection.py:130-162)."""
    A = P.A
    tol = P.tol if tol is None else tol
    if P.tall:
        z0 = np.zeros(A.shape[1]) if x_warm is None else np.asarray(x_warm, float)
        z, it, ok = cgls(lambda t: A @ t, lambda t: A.T @ t, d, c, z0, tol, P.max_inner)
        return z, A @ z, it, ok
    z0 = np.zeros(A.shape[0]) if y_warm is None else np.asarray(y_warm, float) - d
    z, it, ok = cgls(lambda t: A.T @ t, lambda t: A @ t, c, -d, z0, tol, P.max_inner)
    return c - A.T @ z, d + z, it, ok


# -------------------------------------------------------------- solver ----
DEFAULTS = dict(rho0=1.0, abs_tol=1e-4, rel_tol=1e-3, max_iter=10_000,
                alpha=1.7, adaptive_rho=True, delta=1.05, tau=0.8,
                equilibrate=True, projection="direct", projection_tol=None,
                max_inner=None, gap_stop=False)


def prepare(A, settings=None, scaling=None):
    """Equilibrate + rescale + scale + projector (solver.py:148-169)."""
    s = dict(DEFAULTS, **(settings or {}))
    A = np.asarray(A, float)
    m, n = A.shape
    info = dict(iterations=0, converged=True)
    if scaling is not None:
        d, e = scaling
    elif s["equilibrate"]:
        eq = equilibrate(A)
        d, e = rescale_even(A, eq["d"], eq["e"])
        info = dict(iterations=eq["iterations"], converged=eq["converged"])
    else:
        d, e = np.ones(m), np.ones(n)
    Ahat = (d[:, None] * A) * e[None, :]
    tol = s["projection_tol"] if s["projection_tol"] is not None else 1e-8
    P = build_projector(Ahat, tol=tol, max_inner=s["max_inner"],
                        direct=s["projection"] == "direct")
    return dict(d=d, e=e, Ahat=Ahat, P=P, equil=info)


def solve(A, f: Terms, g: Terms, settings=None, x0=None, nu0=None,
          setup=None, callback: Optional[Callable] = None, trace=None):
    """ADMM graph projection splitting (solver.py:248-437).

    Returns a dict with x, y, mu, nu (half iterate, original variables),
    objective, r_pri, r_dual, status ("Solved" / "MaxIterations" /
    "Degenerate"), iterations, final_rho, history (per-iteration
    r_pri, r_dual, eps_pri, eps_dual, rho, objective) and the setup.
    """
    s = dict(DEFAULTS, **(settings or {}))
    A = np.asarray(A, float)
    m, n = A.shape
    if setup is None:
        setup = prepare(A, s)
    d, e, Ahat, P = setup["d"], setup["e"], setup["Ahat"], setup["P"]
    rho = float(s["rho0"])
    alpha = s["alpha"]
    xk, yk, xt, yt = np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(m)
    if x0 is not None:
        xk = np.asarray(x0, float) / e
        yk = Ahat @ xk
    if nu0 is not None:
        nh0 = np.asarray(nu0, float) / d
        yt = -nh0 / rho
        xt = (Ahat.T @ nh0) / rho
    lo_mark = up_mark = 0
    status, iters = "MaxIterations", s["max_iter"]
    xh, yh, muh, nuh = np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(m)
    obj = evaluate(f, yh) + evaluate(g, xh)
    r_pri = r_dual = float("inf")
    gap = None
    hist = []
    indirect = s["projection"] == "indirect"
    for k in range(s["max_iter"]):
        px = prox(g, rho / (e * e), e * (xk - xt))
        py = prox(f, rho * d * d, (yk - yt) / d)
        if not (np.all(np.isfinite(px)) and np.all(np.isfinite(py))):
            status, iters = "Degenerate", k
            break
        xh, yh = px, py
        xhh, yhh = xh / e, yh * d                       # hat-space half iterate
        muh = (-rho * (xhh - xk + xt)) / e              # recover_duals + unscale
        nuh = d * (-rho * (yhh - yk + yt))
        r_pri = float(np.linalg.norm(A @ xh - yh))      # residual_stop
        r_dual = float(np.linalg.norm(A.T @ nuh + muh))
        eps_pri = s["abs_tol"] + s["rel_tol"] * float(np.linalg.norm(yh))
        eps_dual = s["abs_tol"] + s["rel_tol"] * float(np.linalg.norm(muh))
        obj = evaluate(f, yh) + evaluate(g, xh)
        hist.append((r_pri, r_dual, eps_pri, eps_dual, rho, obj))
        if callback is not None:
            callback(k, r_pri, r_dual, eps_pri, eps_dual, rho, obj)
        if trace is not None:
            trace.append(dict(k=k, rho=rho, x_hat=xk.copy(), y_hat=yk.copy(),
                              xt=xt.copy(), yt=yt.copy(), x_half_hat=xhh.copy(),
                              y_half_hat=yhh.copy(), inner_iterations=0))
        if r_pri <= eps_pri and r_dual <= eps_dual:
            status, iters = "Solved", k + 1
            break
        if s["gap_stop"]:                                # solver.py:378-390
            xf, yf = e * xk, yk / d
            muf, nuf = -rho * xt / e, -rho * d * yt
            gap = duality_gap(f, g, xf, yf, muf, nuf)
            if gap is not None and np.isfinite(gap):
                objf = evaluate(f, yf) + evaluate(g, xf)
                if np.isfinite(objf) and gap <= s["abs_tol"] + s["rel_tol"] * abs(objf):
                    status, iters = "Solved", k + 1
                    break
        rx = alpha * xhh + (1.0 - alpha) * xk
        ry = alpha * yhh + (1.0 - alpha) * yk
        cx, cy = rx + xt, ry + yt
        if indirect:
            if s["projection_tol"] is not None:
                ptol = s["projection_tol"]
            else:
                drift = np.sqrt(float(np.sum((xhh - xk) ** 2)) + float(np.sum((yhh - yk) ** 2)))
                ptol = min(1e-2, max(1e-10, 0.1 * drift))
            xn, yn, inner, _ = project_indirect(P, cx, cy, xk, yk, tol=ptol)
            if trace is not None:
                trace[-1]["inner_iterations"] = inner
        else:
            xn, yn = project(P, cx, cy)
        if not (np.all(np.isfinite(xn)) and np.all(np.isfinite(yn))):
            status, iters = "Degenerate", k + 1
            break
        xt = xt + rx - xn
        yt = yt + ry - yn
        xk, yk = xn, yn
        if s["adaptive_rho"]:                            # adapt_rho, Alg. 3
            if r_dual < eps_dual and s["tau"] * k > lo_mark:
                new = s["delta"] * rho
                ratio = rho / new
                rho, up_mark = new, k
                xt, yt = xt * ratio, yt * ratio
            elif r_pri < eps_pri and s["tau"] * k > up_mark:
                new = rho / s["delta"]
                ratio = rho / new
                rho, lo_mark = new, k
                xt, yt = xt * ratio, yt * ratio
    return dict(x=xh, y=yh, mu=muh, nu=nuh, objective=obj, r_pri=r_pri,
                r_dual=r_dual, status=status, iterations=iters, final_rho=rho, gap=gap,
                history=np.array(hist, float).reshape(-1, 6), setup=setup)

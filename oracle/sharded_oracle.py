"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Row-partitioned restatement of ``graphform_oracle.solve`` (the schedule the
CUDA library runs under a communicator, see
``paper_1503_08366_b200/distributed.py`` and DESIGN.md "Multi-GPU").  Each
rank holds rows [r0, r1) of A and f; every cross-row quantity goes through
the caller's ``allreduce(np.ndarray) -> np.ndarray`` (sum), in the SAME
payloads the device issues:

  Sinkhorn sweep   [ sum_i d_i A_ij^2 (n) | ||d - d_old||^2 ]
  rescale          [ ||D A E||_F^2 ]
  projector        I + sum_r A_r' A_r           (n x n, once)
  iteration        [ A_hat' c_y (n) | A' nu_half (n) |
                     ||A x_half - y_half||^2, ||y_half||^2, f(y_half),
                     ||y_half_hat - y_hat||^2, f(y_full), f*(nu_full) ]
                   (one all-reduce; the last two only with gap_stop)
  indirect CGLS    A_hat' r and the m-length dot products

so a world-size-2 ``gloo`` run on CPU checks that the decomposition
reproduces the single-process algorithm (and hence the reference goldens).
Only ``tests/`` imports this module.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from . import graphform_oracle as orc


def equilibrate(A_loc, m_glob, allreduce, max_iter=300):
    """equilibration.py:134-197 over a row partition (gamma/eps use the global m)."""
    m, n = m_glob, A_loc.shape[1]
    gamma = (m + n) * np.sqrt(np.finfo(float).eps)
    eps = 1e-4 * np.sqrt(max(m, n))
    e_it = np.ones(n)
    d_old = None
    done = False
    sweeps = 0
    while sweeps < max_iter:
        sweeps += 1
        d_it = n / (orc._sq_rows(A_loc, e_it) + gamma / m)
        moved_d2 = 0.0 if d_old is None else float(np.sum((d_it - d_old) ** 2))
        red = allreduce(np.concatenate([orc._sq_cols(A_loc, d_it), [moved_d2]]))
        e_next = m / (red[:n] + gamma / n)
        moved_e = np.linalg.norm(e_next - e_it)
        e_it = e_next
        if d_old is not None and moved_e <= eps and np.sqrt(red[n]) <= eps:
            done = True
            break
        d_old = d_it
    return np.sqrt(d_it), np.sqrt(e_it), sweeps, done


def rescale_even(A_loc, m_glob, d, e, allreduce):
    """equilibration.py:200-224 with the Frobenius norm summed over ranks."""
    fro2 = allreduce(np.array([float((d * d) @ orc._sq_rows(A_loc, e * e))]))[0]
    s = np.sqrt(np.sqrt(fro2) / np.sqrt(min(m_glob, A_loc.shape[1])))
    return d / s, e / s


def _cgls(A_loc, allreduce, h1, h2, z0, tol, max_inner):
    """projection.py:165-196, tall: G = A_hat (rows split), z replicated."""
    dot_m = lambda u, v: float(allreduce(np.array([float(u @ v)]))[0])
    rmv = lambda r: allreduce(A_loc.T @ r)
    z = np.array(z0, float, copy=True)
    r1 = h1 - A_loc @ z
    r2 = h2 - z
    s = rmv(r1) + r2
    gam = float(s @ s)
    ref = float(np.linalg.norm(rmv(h1) + h2)) or 1.0
    thr = (tol * ref) ** 2
    if gam <= thr:
        return z, 0
    p = s.copy()
    for it in range(1, max_inner + 1):
        q = A_loc @ p
        den = dot_m(q, q) + float(p @ p)
        if den <= 0.0 or not np.isfinite(den):
            return z, it
        step = gam / den
        z += step * p
        r1 -= step * q
        r2 -= step * p
        s = rmv(r1) + r2
        gnew = float(s @ s)
        if gnew <= thr:
            return z, it
        p = s + (gnew / gam) * p
        gam = gnew
    return z, max_inner


def solve(A_loc, f_loc: orc.Terms, g: orc.Terms, m_glob, allreduce, settings=None):
    """graphform_oracle.solve over this rank's rows.  Returns x, mu (full),
    y, nu (local rows), iterations, status, history like the oracle."""
    s = dict(orc.DEFAULTS, **(settings or {}))
    A_loc = np.asarray(A_loc, float)
    n = A_loc.shape[1]
    if m_glob < n:
        raise ValueError("row-partitioned solves require a tall matrix")
    if s["equilibrate"]:
        d, e, _, _ = equilibrate(A_loc, m_glob, allreduce)
        d, e = rescale_even(A_loc, m_glob, d, e, allreduce)
    else:
        d, e = np.ones(A_loc.shape[0]), np.ones(n)
    Ah = (d[:, None] * A_loc) * e[None, :]
    indirect = s["projection"] == "indirect"
    max_inner = s["max_inner"] if s["max_inner"] is not None else max(100, 2 * min(m_glob, n))
    if not indirect:
        G = allreduce(Ah.T @ Ah)
        G[np.diag_indices_from(G)] += 1.0
        factor = scipy.linalg.cho_factor(G, lower=True)
    rho, alpha = float(s["rho0"]), s["alpha"]
    xk, xt = np.zeros(n), np.zeros(n)
    yk, yt = np.zeros(A_loc.shape[0]), np.zeros(A_loc.shape[0])
    lo_mark = up_mark = 0
    status, iters = "MaxIterations", s["max_iter"]
    hist = []
    xh = muh = None
    for k in range(s["max_iter"]):
        xh = orc.prox(g, rho / (e * e), e * (xk - xt))
        yh = orc.prox(f_loc, rho * d * d, (yk - yt) / d)
        xhh, yhh = xh / e, yh * d
        muh = (-rho * (xhh - xk + xt)) / e
        nuh = d * (-rho * (yhh - yk + yt))
        rx = alpha * xhh + (1.0 - alpha) * xk
        ry = alpha * yhh + (1.0 - alpha) * yk
        cx, cy = rx + xt, ry + yt
        gy = [0.0, 0.0]
        if s["gap_stop"]:   # full iterate of this rank's rows (solver.py:379-382)
            fc = orc.conjugate(f_loc, -rho * d * yt)
            gy = [orc.evaluate(f_loc, yk / d), np.nan if fc is None else fc]
        red = allreduce(np.concatenate([
            Ah.T @ cy, A_loc.T @ nuh,
            [float(np.sum((A_loc @ xh - yh) ** 2)), float(yh @ yh), orc.evaluate(f_loc, yh),
             float(np.sum((yhh - yk) ** 2))], gy]))
        aty, atnu = red[:n], red[n:2 * n]
        r_pri = float(np.sqrt(red[2 * n]))
        r_dual = float(np.linalg.norm(atnu + muh))
        eps_pri = s["abs_tol"] + s["rel_tol"] * float(np.sqrt(red[2 * n + 1]))
        eps_dual = s["abs_tol"] + s["rel_tol"] * float(np.linalg.norm(muh))
        obj = red[2 * n + 2] + orc.evaluate(g, xh)
        hist.append((r_pri, r_dual, eps_pri, eps_dual, rho, obj))
        if r_pri <= eps_pri and r_dual <= eps_dual:
            status, iters = "Solved", k + 1
            break
        if s["gap_stop"]:
            gc = orc.conjugate(g, -rho * xt / e)
            fyf, fcj = red[2 * n + 4], red[2 * n + 5]
            if gc is not None and not np.isnan(fcj):
                gxf = orc.evaluate(g, e * xk)
                gap = fyf + fcj + gxf + gc
                objf = fyf + gxf
                if np.isfinite(gap) and np.isfinite(objf) and gap <= s["abs_tol"] + s["rel_tol"] * abs(objf):
                    status, iters = "Solved", k + 1
                    break
        if indirect:
            if s["projection_tol"] is not None:
                ptol = s["projection_tol"]
            else:
                drift = np.sqrt(float(np.sum((xhh - xk) ** 2)) + red[2 * n + 3])
                ptol = min(1e-2, max(1e-10, 0.1 * drift))
            xn, _ = _cgls(Ah, allreduce, cy, cx, xk, ptol, max_inner)
        else:
            xn = scipy.linalg.cho_solve(factor, cx + aty)
        yn = Ah @ xn
        xt = xt + rx - xn
        yt = yt + ry - yn
        xk, yk = xn, yn
        if s["adaptive_rho"]:
            if r_dual < eps_dual and s["tau"] * k > lo_mark:
                new = s["delta"] * rho
                ratio, rho, up_mark = rho / new, new, k
                xt, yt = xt * ratio, yt * ratio
            elif r_pri < eps_pri and s["tau"] * k > up_mark:
                new = rho / s["delta"]
                ratio, rho, lo_mark = rho / new, new, k
                xt, yt = xt * ratio, yt * ratio
    return dict(x=xh, y=yh, mu=muh, nu=nuh, iterations=iters, status=status,
                history=np.array(hist, float).reshape(-1, 6), d=d, e=e)

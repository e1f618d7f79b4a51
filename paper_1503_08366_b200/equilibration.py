"""Sinkhorn-Knopp equilibration on the GPU (reference equilibration.py).

``equilibrate`` and ``rescale_even`` keep the reference signatures, defaults
and error types (equilibration.py:134-224); the sweeps run as fused
row/column sum-of-squares reductions in fp64 (csrc/gf_equil.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Callable, Optional

import ctypes as C
import numpy as np

from . import _native
from .errors import DimensionError, ParameterError

__all__ = ["Equilibration", "EquilibrationReport", "equilibrate", "rescale_even", "check_equilibrated",
           "equilibration_objective"]


@dataclass(frozen=True)
class Equilibration:
    """Diagonals d = diag(D), e = diag(E) with bookkeeping
    (equilibration.py:38-61)."""

    d: np.ndarray
    e: np.ndarray
    p: int = 2
    gamma: float = 0.0
    iterations: int = 0
    converged: bool = True

    def __post_init__(self):
        d = np.asarray(self.d, dtype=float)
        e = np.asarray(self.e, dtype=float)
        object.__setattr__(self, "d", d)
        object.__setattr__(self, "e", e)
        if not (np.all(d > 0.0) and np.all(np.isfinite(d))):
            raise ParameterError("diagonal d must be positive and finite")
        if not (np.all(e > 0.0) and np.all(np.isfinite(e))):
            raise ParameterError("diagonal e must be positive and finite")

    @classmethod
    def identity(cls, m: int, n: int) -> "Equilibration":
        return cls(d=np.ones(m), e=np.ones(n))


def _matrix_dtype(A):
    # fp64 like the reference (equilibration.py:150 works on float64 A),
    # whatever the input's storage type
    return _native.GF_F64


def _as_matrix(A):
    if _native.is_torch(A):
        if A.dim() != 2:
            raise ParameterError("A must be a 2-D matrix")
        return A
    A = np.asarray(A)
    if A.dtype != np.float32:
        A = A.astype(np.float64, copy=False)
    if A.ndim != 2:
        raise ParameterError("A must be a 2-D matrix")
    return A


def equilibrate(A, gamma: Optional[float] = None, eps: Optional[float] = None,
                max_iter: int = 300, on_sweep: Optional[Callable] = None) -> Equilibration:
    """Regularised Sinkhorn-Knopp with p = 2 (equilibration.py:134-197).
    ``on_sweep(k, d, e)`` receives the diagonal iterates after each sweep
    (host copies made by the library after the sweep's device updates); an
    exception it raises is re-raised once the sweeps return."""
    A = _as_matrix(A)
    if gamma is not None and gamma < 0.0:
        raise ParameterError("gamma must be nonnegative")
    if eps is not None and not eps > 0.0:
        raise ParameterError("eps must be positive")
    if max_iter < 1:
        raise ParameterError("max_iter must be at least 1")
    L = _native.lib()
    M = _native.Matrix(A, _matrix_dtype(A))
    m, n = M.m, M.n
    d = np.empty(m)
    e = np.empty(n)
    sweeps = C.c_int64()
    conv = C.c_int()
    g_used = C.c_double()
    errors = []

    def observe(k, dp, ep, mm, nn, _user):
        if errors:
            return
        try:
            on_sweep(int(k), np.ctypeslib.as_array(dp, shape=(mm,)).copy(),
                     np.ctypeslib.as_array(ep, shape=(nn,)).copy())
        except BaseException as exc:   # re-raised after the C call returns
            errors.append(exc)

    cb = _native.SWEEP_FN(observe) if on_sweep is not None else None
    _native.check(L.gf_equilibrate_observed(M.handle, -1.0 if gamma is None else float(gamma),
                                            -1.0 if eps is None else float(eps), int(max_iter), None,
                                            _native.ptr(d), _native.ptr(e), C.byref(sweeps), C.byref(conv),
                                            C.byref(g_used), C.cast(cb, C.c_void_p) if cb else None, None,
                                            _native.stream()))
    if errors:
        raise errors[0]
    return Equilibration(d=d, e=e, p=2, gamma=float(g_used.value),
                         iterations=int(sweeps.value), converged=bool(conv.value))


def rescale_even(eq: Equilibration, A) -> Equilibration:
    """Split |DAE|_F / sqrt(min(m, n)) evenly between d and e
    (equilibration.py:214-224)."""
    A = _as_matrix(A)
    m, n = A.shape
    if eq.d.shape != (m,) or eq.e.shape != (n,):
        raise DimensionError(
            f"scaling of lengths {eq.d.shape}/{eq.e.shape} does not match matrix of shape {tuple(A.shape)}")
    L = _native.lib()
    M = _native.Matrix(A, _matrix_dtype(A))
    d = np.array(eq.d, dtype=float, copy=True)
    e = np.array(eq.e, dtype=float, copy=True)
    _native.check(L.gf_rescale_even(M.handle, _native.ptr(d), _native.ptr(e), None, _native.stream()))
    return replace(eq, d=d, e=e)


@dataclass(frozen=True)
class EquilibrationReport:
    """How far DAE is from equilibrated (equilibration.py:64-91)."""

    row_deviation: float        # max relative deviation of row |DAE|^p sums
    col_deviation: float
    identity_abs: float         # |mean(d) - mean(e)|
    identity_rel: float
    frobenius_ratio: float      # |DAE|_F / sqrt(min(m, n))
    tol: float

    @property
    def rows_ok(self) -> bool:
        return self.row_deviation <= self.tol

    @property
    def cols_ok(self) -> bool:
        return self.col_deviation <= self.tol

    def as_dict(self) -> dict:
        return {"row_deviation": self.row_deviation, "col_deviation": self.col_deviation,
                "identity_abs": self.identity_abs, "identity_rel": self.identity_rel,
                "frobenius_ratio": self.frobenius_ratio, "tol": self.tol,
                "rows_ok": self.rows_ok, "cols_ok": self.cols_ok}


def _sq_ops(A):
    """(A o A) x and (A o A)' x on the device (gf_sq_matvec): the p = 2 handles
    of equilibration.py:94-125."""
    L = _native.lib()
    M = _native.Matrix(_as_matrix(A), _matrix_dtype(A))
    m, n = M.m, M.n

    def row_apply(x):
        x = np.ascontiguousarray(x, dtype=float)
        y = np.empty(m)
        _native.check(L.gf_sq_matvec(M.handle, 0, _native.ptr(x), _native.ptr(y), _native.stream()))
        return y

    def col_apply(x):
        x = np.ascontiguousarray(x, dtype=float)
        y = np.empty(n)
        _native.check(L.gf_sq_matvec(M.handle, 1, _native.ptr(x), _native.ptr(y), _native.stream()))
        return y

    return row_apply, col_apply, M


def _check_p(p):
    if p != 2:
        raise ParameterError("the GPU build implements the p = 2 equilibration (as equilibrate does)")


def _check_scaling_dims(A, d, e):
    m, n = A.shape
    if d.shape != (m,) or e.shape != (n,):
        raise DimensionError(
            f"scaling of lengths {d.shape}/{e.shape} does not match matrix of shape {tuple(A.shape)}")


def _max_rel_deviation(sums):   # equilibration.py:263-267
    mean = float(np.mean(sums))
    if mean <= 0.0 or not np.isfinite(mean):
        return float("inf")
    return float(np.max(np.abs(sums - mean)) / mean)


def check_equilibrated(A, d, e, p: int = 2, tol: float = 1e-2) -> EquilibrationReport:
    """Report how far DAE is from equilibrated (equilibration.py:227-267):
    max relative deviations of the row / column sums of |DAE|^p from their
    mean, the identity residual |mean(d) - mean(e)| and |DAE|_F / sqrt(min(m, n))."""
    _check_p(p)
    A = _as_matrix(A)
    m, n = A.shape
    d = np.asarray(d, dtype=float)
    e = np.asarray(e, dtype=float)
    _check_scaling_dims(A, d, e)
    row_apply, col_apply, _M = _sq_ops(A)
    row_sums = (d ** p) * row_apply(e ** p)
    col_sums = (e ** p) * col_apply(d ** p)
    mean_d = float(np.mean(d))
    mean_e = float(np.mean(e))
    identity_abs = abs(mean_d - mean_e)
    identity_rel = identity_abs / max(mean_d, mean_e, np.finfo(float).tiny)
    fro_sq = float(np.sum(row_sums))
    return EquilibrationReport(row_deviation=_max_rel_deviation(row_sums),
                               col_deviation=_max_rel_deviation(col_sums),
                               identity_abs=identity_abs, identity_rel=identity_rel,
                               frobenius_ratio=float(np.sqrt(fro_sq / min(m, n))), tol=float(tol))


def equilibration_objective(A, d, e, gamma: float, p: int = 2) -> float:
    """Regularised scaling objective at diagonals d, e (equilibration.py:270-287):
    d^p' |A|^p e^p - n sum log d^p - m sum log e^p + gamma (sum d^p / m + sum e^p / n)."""
    _check_p(p)
    A = _as_matrix(A)
    m, n = A.shape
    d = np.asarray(d, dtype=float)
    e = np.asarray(e, dtype=float)
    row_apply, _, _M = _sq_ops(A)
    dp = d ** p
    ep = e ** p
    total = float(dp @ row_apply(ep))
    total -= n * float(np.sum(np.log(dp)))
    total -= m * float(np.sum(np.log(ep)))
    total += gamma * (float(np.sum(dp)) / m + float(np.sum(ep)) / n)
    return total

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

__all__ = ["Equilibration", "equilibrate", "rescale_even"]


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
    return _native.GF_F32 if str(getattr(A, "dtype", "")).endswith("float32") else _native.GF_F64


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
    """Regularised Sinkhorn-Knopp with p = 2 (equilibration.py:134-197)."""
    if on_sweep is not None:
        raise NotImplementedError("on_sweep callbacks are not supported by the GPU build")
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
    _native.check(L.gf_equilibrate(M.handle, -1.0 if gamma is None else float(gamma),
                                   -1.0 if eps is None else float(eps), int(max_iter), None,
                                   _native.ptr(d), _native.ptr(e), C.byref(sweeps), C.byref(conv),
                                   C.byref(g_used), _native.stream()))
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

"""Graph projection on the GPU (reference projection.py).

``build_projector`` forms I + A'A (m >= n) or I + AA' (m < n) on the device,
factors it (blocked Cholesky, fp64) and keeps the explicit inverse that the
per-iteration apply streams as one GEMV (csrc/gf_dense.cu); ``project`` is the
reduced update of projection.py:112-127.  ``BUILD_COUNT`` counts builds in
this process (projection.py:29, SPEC acceptance criterion 8).
"""

from __future__ import annotations

from typing import NamedTuple, Optional

import ctypes as C
import numpy as np

from . import _native
from .errors import DimensionError, ParameterError

__all__ = ["ProjectorCache", "IndirectResult", "build_projector", "project", "project_indirect"]

BUILD_COUNT = 0


class IndirectResult(NamedTuple):
    x: np.ndarray
    y: np.ndarray
    iterations: int
    converged: bool


class ProjectorCache:
    """Handle of a device-side projector (projection.py:39-49).

    ``gram`` is fetched from the device on first access; ``chol`` is None
    (the factor never leaves the device)."""

    def __init__(self, handle, matrix, mode, m, n, tol, max_inner, owner=None):
        self.handle = handle
        self._matrix = matrix      # keeps the gf_matrix alive
        self._owner = owner        # Setup that owns handle, if any
        self.mode = mode
        self.m, self.n = m, n
        self.orientation = "tall" if m >= n else "wide"
        self.tol = float(tol)
        self.max_inner = int(max_inner)
        self.chol = None
        self._gram = None

    @property
    def A(self):
        return self._matrix.download() if self._matrix is not None else None

    @property
    def gram(self):
        if self.mode != "direct":
            return None
        if self._gram is None:
            q = min(self.m, self.n)
            g = np.empty((q, q))
            _native.check(_native.lib().gf_projector_gram(self.handle, _native.ptr(g), _native.stream()))
            self._gram = g
        return self._gram

    def __del__(self):
        try:
            if self._owner is None and self.handle:
                _native.load_library().gf_projector_destroy(self.handle)
        except Exception:
            pass


def build_projector(A, mode: str = "direct", tol: float = 1e-8,
                    max_inner: Optional[int] = None, precision: Optional[str] = None) -> ProjectorCache:
    """Prepare the projection onto the graph of ``A`` (projection.py:61-99)."""
    global BUILD_COUNT
    if mode not in ("direct", "indirect"):
        raise ParameterError(f"unknown projection mode {mode!r}")
    if not tol > 0.0:
        raise ParameterError("projection tolerance must be positive")
    if hasattr(A, "nnz") and hasattr(A, "tocsr"):
        raise ParameterError("sparse matrices are not supported by the GPU build")
    if not _native.is_torch(A):
        A = np.asarray(A)
        if A.dtype != np.float32:
            A = A.astype(np.float64, copy=False)
    if A.ndim != 2:
        raise DimensionError("A must be a 2-D matrix")
    m, n = int(A.shape[0]), int(A.shape[1])
    if max_inner is None:
        max_inner = max(100, 2 * min(m, n))
    dt = _dtype_for(A, precision)
    L = _native.lib()
    M = _native.Matrix(A, dt)
    h = C.c_void_p()
    _native.check(L.gf_projector_create(M.handle, 0 if mode == "direct" else 1, float(tol), int(max_inner),
                                        None, _native.stream(), C.byref(h)))
    BUILD_COUNT += 1
    return ProjectorCache(h, M, mode, m, n, tol, max_inner)


def _dtype_for(A, precision):
    # the reference coerces every input to float64 (problem.py:35); fp32
    # arithmetic is opt-in only
    if precision is None:
        return _native.GF_F64
    if precision in ("fp32", "float32"):
        return _native.GF_F32
    if precision in ("fp64", "float64"):
        return _native.GF_F64
    raise ParameterError(f"unknown precision {precision!r}")


def _check_query(cache, c, d):
    c = np.asarray(c, dtype=float)
    d = np.asarray(d, dtype=float)
    if c.shape != (cache.n,) or d.shape != (cache.m,):
        raise DimensionError(f"expected c of length {cache.n} and d of length {cache.m}")
    return np.ascontiguousarray(c), np.ascontiguousarray(d)


def project(cache: ProjectorCache, c, d):
    """Exact projection of (c, d) onto {(x, y): y = A x} (projection.py:112-127)."""
    if cache.mode != "direct":
        raise ParameterError("project requires a direct-mode cache; use project_indirect")
    c, d = _check_query(cache, c, d)
    x = np.empty(cache.n)
    y = np.empty(cache.m)
    _native.check(_native.lib().gf_project(cache.handle, _native.ptr(c), _native.ptr(d), _native.ptr(x),
                                           _native.ptr(y), _native.stream()))
    return x, y


def project_indirect(cache: ProjectorCache, c, d, x_warm=None, y_warm=None,
                     tol: Optional[float] = None) -> IndirectResult:
    """CGLS projection (projection.py:130-162)."""
    c, d = _check_query(cache, c, d)
    if tol is None:
        tol = cache.tol
    if not tol > 0.0:
        raise ParameterError("projection tolerance must be positive")
    x = np.empty(cache.n)
    y = np.empty(cache.m)
    xw = None if x_warm is None else np.ascontiguousarray(np.asarray(x_warm, float))
    yw = None if y_warm is None else np.ascontiguousarray(np.asarray(y_warm, float))
    it = C.c_int64()
    ok = C.c_int()
    _native.check(_native.lib().gf_project_indirect(
        cache.handle, _native.ptr(c), _native.ptr(d), None if xw is None else _native.ptr(xw),
        None if yw is None else _native.ptr(yw), float(tol), _native.ptr(x), _native.ptr(y),
        C.byref(it), C.byref(ok), _native.stream()))
    return IndirectResult(x=x, y=y, iterations=int(it.value), converged=bool(ok.value))

"""Separable objectives c*h(a*x - b) + d*x + (e/2)*x**2 (host-side model).

Mirrors the reference function model (``functions.py``): ten base kinds whose
integer codes follow enum order (``functions.py:34-60``), per-coordinate
term parameters stored as flat arrays (structure of arrays), and the same
validation (a != 0, c >= 0, e >= 0, finite; ``functions.py:215-225``).

Only the data model lives on the host.  Evaluation (``evaluate``,
``eval_base``) runs in the CUDA library (``gf_evaluate`` / ``gf_eval_base``
in ``include/graphform_b200.h``); the per-kind arithmetic is in
``csrc/gf_terms.cuh``.  The device copy of the term arrays is built once per
(function, device) and cached on the instance.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from functools import cached_property
from typing import Iterable

import numpy as np

from .errors import DimensionError, ParameterError

__all__ = ["BaseFunction", "FunctionTerm", "SeparableFunction", "eval_base",
           "conjugate_base", "KIND_CODE", "CODE_KIND"]


class BaseFunction(enum.Enum):
    ABS = "Abs"            # |x|
    SQUARE = "Square"      # x^2 / 2
    HUBER = "Huber"        # x^2/2 on |x| <= 1, |x| - 1/2 outside
    NEG_ENTR = "NegEntr"   # x log x on x >= 0
    LOGISTIC = "Logistic"  # log(1 + e^x)
    MAX_POS0 = "MaxPos0"   # max(0, x)
    IND_GE0 = "IndGe0"     # 0 if x >= 0 else +inf
    IND_LE0 = "IndLe0"     # 0 if x <= 0 else +inf
    IND_EQ0 = "IndEq0"     # 0 if x == 0 else +inf
    ZERO = "Zero"          # 0

    @classmethod
    def from_name(cls, name) -> "BaseFunction":
        """Case- and underscore-insensitive lookup (functions.py:48-57)."""
        hit = _BY_NAME.get(str(name).replace("_", "").lower())
        if hit is None:
            raise ParameterError(f"unknown base function {name!r}")
        return hit


_BY_NAME = {k.value.lower(): k for k in BaseFunction}
CODE_KIND = list(BaseFunction)
KIND_CODE = {k: i for i, k in enumerate(CODE_KIND)}
ZERO_CODE = KIND_CODE[BaseFunction.ZERO]
NUM_KINDS = len(CODE_KIND)


def kind_code(h) -> int:
    if isinstance(h, BaseFunction):
        return KIND_CODE[h]
    if isinstance(h, (int, np.integer)):
        return int(h)
    return KIND_CODE[BaseFunction.from_name(h)]


@dataclass(frozen=True)
class FunctionTerm:
    """One coordinate: ``c*h(a*x - b) + d*x + (e/2)*x**2``."""

    h: BaseFunction
    a: float = 1.0
    b: float = 0.0
    c: float = 1.0
    d: float = 0.0
    e: float = 0.0

    def __post_init__(self):
        for name in ("a", "b", "c", "d", "e"):
            val = float(getattr(self, name))
            if not np.isfinite(val):
                raise ParameterError(f"term parameter {name} must be finite")
            object.__setattr__(self, name, val)
        if not isinstance(self.h, BaseFunction):
            object.__setattr__(self, "h", BaseFunction.from_name(self.h))
        if self.a == 0.0:
            raise ParameterError("term scale a must be nonzero")
        if self.c < 0.0:
            raise ParameterError("term weight c must be nonnegative")
        if self.e < 0.0:
            raise ParameterError("term quadratic e must be nonnegative")


_PARAMS = ("a", "b", "c", "d", "e")


@dataclass(frozen=True, eq=False)
class SeparableFunction:
    """Coordinatewise sum of parametric terms stored as flat arrays."""

    h: np.ndarray
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray
    e: np.ndarray
    _device_cache: dict = field(default_factory=dict, init=False, repr=False,
                                compare=False)

    def __post_init__(self):
        codes = np.asarray(self.h, dtype=np.int64).ravel()
        object.__setattr__(self, "h", codes)
        size = codes.size
        for name in _PARAMS:
            arr = np.asarray(getattr(self, name), dtype=np.float64)
            if arr.ndim == 0:
                arr = np.full(size, float(arr))
            if arr.shape != (size,):
                raise DimensionError(f"parameter array {name} has wrong length")
            object.__setattr__(self, name, arr)
        if size and (codes.min() < 0 or codes.max() >= NUM_KINDS):
            raise ParameterError("invalid base function code")
        for name in _PARAMS:
            if not np.all(np.isfinite(getattr(self, name))):
                raise ParameterError(f"parameter array {name} must be finite")
        if np.any(self.a == 0.0):
            raise ParameterError("term scale a must be nonzero")
        if np.any(self.c < 0.0):
            raise ParameterError("term weight c must be nonnegative")
        if np.any(self.e < 0.0):
            raise ParameterError("term quadratic e must be nonnegative")

    @classmethod
    def from_terms(cls, terms: Iterable[FunctionTerm]) -> "SeparableFunction":
        terms = list(terms)
        cols = {p: np.array([getattr(t, p) for t in terms], dtype=np.float64)
                for p in _PARAMS}
        return cls(h=np.array([KIND_CODE[t.h] for t in terms], dtype=np.int64),
                   **cols)

    @classmethod
    def from_arrays(cls, h, size=None, a=1.0, b=0.0, c=1.0, d=0.0, e=0.0):
        if isinstance(h, (BaseFunction, str)):
            if size is None:
                raise ParameterError("size required when h is a single kind")
            codes = np.full(size, kind_code(h), dtype=np.int64)
        else:
            codes = np.array([kind_code(k) for k in np.ravel(h)], dtype=np.int64)
            if size is not None and codes.size != size:
                raise DimensionError("kind array does not match size")
        return cls(h=codes, a=a, b=b, c=c, d=d, e=e)

    @classmethod
    def uniform(cls, h, size, **params) -> "SeparableFunction":
        return cls.from_arrays(h, size=size, **params)

    def __len__(self) -> int:
        return int(self.h.size)

    @cached_property
    def terms(self) -> tuple:
        return tuple(FunctionTerm(CODE_KIND[int(self.h[i])], a=self.a[i],
                                  b=self.b[i], c=self.c[i], d=self.d[i],
                                  e=self.e[i]) for i in range(len(self)))

    @cached_property
    def _effective(self):
        """(codes, c_eff): c == 0 coordinates act as ZERO with c_eff = 1
        (functions.py:284-303).  The device kernels apply the same rule
        per element; this host view exists for inspection and tests."""
        zero_c = self.c == 0.0
        return (np.where(zero_c, ZERO_CODE, self.h),
                np.where(zero_c, 1.0, self.c))

    def slice(self, start: int, stop: int) -> "SeparableFunction":
        """Coordinates [start, stop) -- the row shard of f under a row
        partition of A (one rank's rows)."""
        return SeparableFunction(self.h[start:stop], *(getattr(self, p)[start:stop]
                                                      for p in _PARAMS))

    def evaluate(self, v) -> float:
        """Sum of all terms at ``v``; +inf when an indicator is violated
        (functions.py:307-327).  Runs on the GPU."""
        from . import _native
        return _native.evaluate(self, v)

    def conjugate(self, w):
        """Coordinatewise conjugate sum, or ``None`` when some term has e > 0
        and a kind whose composition has no closed form (functions.py:329-393).
        Runs on the GPU."""
        from . import _native
        return _native.conjugate(self, w)


def eval_base(h, x):
    """Evaluate base function ``h`` elementwise (+inf off-domain) on the GPU."""
    from . import _native
    return _native.eval_base(kind_code(h), x)


def conjugate_base(h, w):
    """Convex conjugate of base function ``h`` elementwise (functions.py:147-150),
    on the GPU."""
    from . import _native
    return _native.conj_base(kind_code(h), w)

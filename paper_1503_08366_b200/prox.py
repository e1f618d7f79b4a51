"""Separable prox on the GPU (reference prox.py:101-138).

The argument checks and their error types follow the reference exactly; the
arithmetic runs in the CUDA kernels ``gf_prox_separable`` / ``gf_prox_base``
(csrc/gf_terms.cuh), fp64, one thread per coordinate, including the
safeguarded Newton loops of Logistic and NegEntr (prox.py:27-70).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import DimensionError, ParameterError
from .functions import SeparableFunction, kind_code

__all__ = ["prox_base", "prox_separable"]

STATIONARITY_TOL = 1e-12   # prox.py:23 (applied on the device)
MAX_NEWTON_ITER = 100      # prox.py:24


def _check_rho(rho_t):
    import torch
    if not bool(torch.all(rho_t > 0.0)) or not bool(torch.all(torch.isfinite(rho_t))):
        raise ParameterError("prox parameters must be positive and finite")


def prox_base(h, rho, v):
    """Prox of one base function; scalar in, scalar out; arrays broadcast."""
    import torch
    code = kind_code(h)
    scalar = np.ndim(v) == 0 and not _native.is_torch(v)
    v_t = _native.to_device64(np.atleast_1d(np.asarray(v, float)) if scalar else v)
    shape = v_t.shape
    v_t = v_t.reshape(-1)
    rho_t = torch.broadcast_to(_native.to_device64(np.asarray(rho, float) if not _native.is_torch(rho) else rho),
                               shape).reshape(-1).contiguous()
    if not bool(torch.all(rho_t > 0.0)) or not bool(torch.all(torch.isfinite(rho_t))):
        raise ParameterError("prox parameter rho must be positive and finite")
    out = _native.prox_base_dev(code, rho_t, v_t).reshape(shape)
    if scalar:
        return float(out.item())
    return _native.like_input(out, v)


def prox_separable(sf: SeparableFunction, rho, v):
    """Coordinatewise prox of ``sf`` at per-coordinate (or scalar) ``rho``."""
    import torch
    n = len(sf)
    if not _native.is_torch(v):
        vn = np.asarray(v, dtype=float)
        if vn.shape != (n,):
            raise DimensionError(f"expected vector of length {n}, got shape {vn.shape}")
    elif tuple(v.shape) != (n,):
        raise DimensionError(f"expected vector of length {n}, got shape {tuple(v.shape)}")
    v_t = _native.to_device64(v)
    if _native.is_torch(rho):
        rho_t = rho.to(device=v_t.device, dtype=torch.float64)
    else:
        rho_t = _native.to_device64(np.asarray(rho, dtype=float))
    if rho_t.dim() == 0:
        rho_t = rho_t.expand(n)
    elif tuple(rho_t.shape) != (n,):
        raise DimensionError("rho vector does not match function length")
    rho_t = rho_t.contiguous()
    _check_rho(rho_t)
    return _native.like_input(_native.prox_separable_dev(sf, rho_t, v_t), v)

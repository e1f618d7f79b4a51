"""Synthetic instance recipes (host-side input synthesis, not the solve path).

The nine Appendix-A families of the reference, restated so that an instance
built here is bit-identical to the reference's ``generate(GenSpec(...))``
for the same (family, m, n, seed): every array draws from its own PCG64
stream spawned from ``SeedSequence([seed, family_index])`` in a fixed order
(reference ``generators.py:80-84``).  ``tall_lasso`` is the Lasso recipe
without the reference's ``m < n`` guard (``generators.py:146-157``), which the
BASELINE configs need because they are tall.

Everything here is numpy on the host: it builds inputs, it never solves.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError
from .functions import BaseFunction, SeparableFunction
from .problem import GraphFormProblem

__all__ = ["FAMILIES", "GenSpec", "generate", "tall_lasso", "tall_ridge", "canonical_family"]

# Family order fixes the SeedSequence index (generators.py:25-35).
FAMILIES = (
    "basis_pursuit", "entropy_max", "huber_fit", "lasso", "logistic",
    "lp", "nnls", "portfolio", "svm",
)
_INDEX = {name: k for k, name in enumerate(FAMILIES)}
_ALIAS = {
    "basispursuit": "basis_pursuit", "entropymax": "entropy_max",
    "huberfit": "huber_fit", "huber": "huber_fit",
    "logisticregression": "logistic", "linearprogram": "lp",
    "nonnegleastsquares": "nnls", "supportvectormachine": "svm",
}


def canonical_family(name: str) -> str:
    """Family lookup tolerant to case, '-' and '_' (generators.py:51-60)."""
    key = str(name).strip().lower().replace("-", "_")
    if key in _INDEX:
        return key
    flat = key.replace("_", "")
    if flat in _ALIAS:
        return _ALIAS[flat]
    if flat in _INDEX:
        return flat
    raise ParameterError(f"unknown problem family {name!r}")


@dataclass(frozen=True)
class GenSpec:
    family: str
    m: int
    n: int
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "family", canonical_family(self.family))
        if self.m < 1 or self.n < 1:
            raise ParameterError("dimensions must be positive")


def _rngs(family: str, seed: int, count: int):
    root = np.random.SeedSequence([int(seed), _INDEX[family]])
    return [np.random.default_rng(s) for s in root.spawn(count)]


def _need(ok: bool, msg: str):
    if not ok:
        raise ParameterError(msg)


def _plant(rng, n):
    coef = rng.normal(0.0, 1.0 / np.sqrt(n), size=n)
    coef[rng.random(n) < 0.5] = 0.0
    return coef


def _lasso_arrays(m, n, seed):
    r_a, r_v, r_n = _rngs("lasso", seed, 3)
    A = r_a.normal(size=(m, n))
    v = _plant(r_v, n)
    b = A @ v + r_n.normal(0.0, 0.5, size=m)
    lam = 0.2 * float(np.max(np.abs(A.T @ b)))
    return A, v, b, lam


def tall_lasso(m: int, n: int, seed: int = 0, dtype=np.float64, device: bool = False):
    """Lasso with any aspect ratio: f = Square(b), g = lam*Abs.

    ``dtype=np.float32`` rounds A, b and lam to fp32 and returns them as
    float64 arrays holding fp32 values (the fp32 parity protocol: the GPU and
    the CPU oracle see the same rounded numbers).  ``device=True`` draws A on
    the GPU (bit-identical to the host stream) and returns it as a CUDA tensor.
    """
    if device:
        return _dev_tall_lasso(m, n, seed, dtype)
    A, v, b, lam = _lasso_arrays(m, n, seed)
    if np.dtype(dtype) == np.float32:
        A = A.astype(np.float32)
        b = b.astype(np.float32).astype(np.float64)
        lam = float(np.float32(lam))
    f = SeparableFunction.from_arrays(BaseFunction.SQUARE, size=m, b=b)
    g = SeparableFunction.from_arrays(BaseFunction.ABS, size=n, c=lam)
    return GraphFormProblem(A, f, g), {"v": v, "b": b, "lam": lam}


def tall_ridge(m: int, n: int, seed: int = 0, dtype=np.float64):
    """tall_lasso's data with g = lam * Square (every conjugate finite: the
    duality gap is a usable stopping rule; test fixture family)."""
    problem, meta = tall_lasso(m, n, seed, dtype)
    g = SeparableFunction.from_arrays(BaseFunction.SQUARE, size=n, c=meta["lam"])
    return GraphFormProblem(problem.A, problem.f, g), meta


def _gen_lasso(s):
    _need(s.m < s.n, "lasso needs m < n")
    A, v, b, lam = _lasso_arrays(s.m, s.n, s.seed)
    f = SeparableFunction.from_arrays(BaseFunction.SQUARE, size=s.m, b=b)
    g = SeparableFunction.from_arrays(BaseFunction.ABS, size=s.n, c=lam)
    return GraphFormProblem(A, f, g), {"v": v, "b": b, "lam": lam}


def _gen_basis_pursuit(s):
    _need(s.m > s.n, "basis_pursuit needs m > n")
    r_a, r_v = _rngs(s.family, s.seed, 2)
    A = r_a.normal(size=(s.m, s.n))
    v = _plant(r_v, s.n)
    b = A @ v
    f = SeparableFunction.from_arrays(BaseFunction.IND_EQ0, size=s.m, b=b)
    g = SeparableFunction.uniform(BaseFunction.ABS, s.n)
    return GraphFormProblem(A, f, g), {"v": v, "b": b}


def _gen_entropy_max(s):
    _need(s.m < s.n, "entropy_max needs m < n")
    r_a, r_v = _rngs(s.family, s.seed, 2)
    A0 = r_a.normal(0.0, np.sqrt(s.n), size=(s.m, s.n))
    v = r_v.random(s.n)
    b = (A0 @ v) / v.sum()
    A = np.vstack([A0, np.ones((1, s.n))])
    f = SeparableFunction.from_arrays(
        [BaseFunction.IND_LE0] * s.m + [BaseFunction.IND_EQ0],
        b=np.concatenate([b, [1.0]]))
    g = SeparableFunction.uniform(BaseFunction.NEG_ENTR, s.n)
    return GraphFormProblem(A, f, g), {"v": v, "b": b}


def _gen_huber_fit(s):
    _need(s.m > s.n, "huber_fit needs m > n")
    r_a, r_v, r_e, r_o = _rngs(s.family, s.seed, 4)
    A = r_a.normal(0.0, np.sqrt(s.n), size=(s.m, s.n))
    v = r_v.normal(0.0, 1.0 / np.sqrt(s.n), size=s.n)
    noise = r_e.normal(0.0, 0.5, size=s.m)
    out = r_o.random(s.m) >= 0.95
    noise[out] = r_o.random(out.sum()) * 10.0
    b = A @ v + noise
    f = SeparableFunction.from_arrays(BaseFunction.HUBER, size=s.m, b=b)
    g = SeparableFunction.uniform(BaseFunction.ZERO, s.n)
    return GraphFormProblem(A, f, g), {"v": v, "b": b, "outlier_mask": out}


def _gen_logistic(s):
    _need(s.m > s.n, "logistic needs m > n")
    r_a, r_v, r_l = _rngs(s.family, s.seed, 3)
    A = r_a.normal(size=(s.m, s.n))
    v = _plant(r_v, s.n)
    p0 = 1.0 / (1.0 + np.exp(-(A @ v)))
    lab = np.where(r_l.random(s.m) < p0, 0.0, 1.0)
    lam = 0.1 * float(np.max(np.abs(A.T @ (0.5 - lab))))
    f = SeparableFunction.from_arrays(BaseFunction.LOGISTIC, size=s.m, d=-lab)
    g = SeparableFunction.from_arrays(BaseFunction.ABS, size=s.n, c=lam)
    return GraphFormProblem(A, f, g), {"v": v, "labels": lab, "lam": lam}


def _gen_lp(s):
    _need(s.m > s.n, "lp needs m > n")
    r_a, r_v, r_e, r_u = _rngs(s.family, s.seed, 4)
    A = r_a.normal(size=(s.m, s.n))
    v = r_v.normal(0.0, 1.0 / np.sqrt(s.n), size=s.n)
    b = A @ v + r_e.random(s.m) * 0.1
    u = r_u.random(s.m)
    c = -A.T @ u
    f = SeparableFunction.from_arrays(BaseFunction.IND_LE0, size=s.m, b=b)
    g = SeparableFunction.from_arrays(BaseFunction.ZERO, size=s.n, d=c)
    return GraphFormProblem(A, f, g), {"v": v, "u": u, "b": b, "c": c}


def _gen_nnls(s):
    _need(s.m > s.n, "nnls needs m > n")
    r_a, r_v, r_e = _rngs(s.family, s.seed, 3)
    A = r_a.normal(size=(s.m, s.n))
    v = r_v.normal(1.0 / s.n, 1.0 / np.sqrt(s.n), size=s.n)
    b = A @ v + r_e.normal(0.0, 0.5, size=s.m)
    f = SeparableFunction.from_arrays(BaseFunction.SQUARE, size=s.m, b=b)
    g = SeparableFunction.uniform(BaseFunction.IND_GE0, s.n)
    return GraphFormProblem(A, f, g), {"v": v, "b": b}


def _gen_portfolio(s):
    k, n = s.m, s.n
    _need(n > k, "portfolio needs n > k (pass the factor count as m)")
    r_f, r_d, r_mu = _rngs(s.family, s.seed, 3)
    F = r_f.normal(size=(n, k))
    D = r_d.random(n) * np.sqrt(k)
    mu = r_mu.normal(size=n)
    A = np.vstack([F.T, np.ones((1, n))])
    f = SeparableFunction.from_arrays(
        [BaseFunction.ZERO] * k + [BaseFunction.IND_EQ0],
        b=np.concatenate([np.zeros(k), [1.0]]),
        e=np.concatenate([np.full(k, 2.0), [0.0]]))
    g = SeparableFunction.from_arrays(BaseFunction.IND_GE0, size=n, d=-mu, e=2.0 * D)
    return GraphFormProblem(A, f, g), {"D": D, "mu": mu, "gamma_risk": 1.0}


def _gen_svm(s):
    _need(s.m > s.n, "svm needs m > n")
    (r_a,) = _rngs(s.family, s.seed, 1)
    lab = np.where(np.arange(s.m) < s.m // 2, 1.0, -1.0)
    A = r_a.normal(0.0, 1.0 / np.sqrt(s.n), size=(s.m, s.n)) + (lab / s.n)[:, None]
    f = SeparableFunction.from_arrays(BaseFunction.MAX_POS0, size=s.m, b=-1.0, c=1.0)
    g = SeparableFunction.from_arrays(BaseFunction.ZERO, size=s.n, e=2.0)
    return GraphFormProblem(lab[:, None] * A, f, g), {"labels": lab, "lam": 1.0, "raw_A": A}


_BUILD = {
    "basis_pursuit": _gen_basis_pursuit, "entropy_max": _gen_entropy_max,
    "huber_fit": _gen_huber_fit, "lasso": _gen_lasso, "logistic": _gen_logistic,
    "lp": _gen_lp, "nnls": _gen_nnls, "portfolio": _gen_portfolio, "svm": _gen_svm,
}


# ------------------------------------------------- on-device synthesis ----
# the big matrix of every family is drawn on the GPU from
# the same PCG64 stream the host generator uses (gf_normal_fill reproduces
# numpy's normals bit for bit), so A is identical to the reference's; the
# O(m + n) vectors come from the host streams as before, and the products
# A @ v, A.T @ b run on the device in fp64 (their last bits can differ from
# numpy's BLAS, as any change of summation order does).
def _dev_matrix(m, n, dtype=None):
    """Zeroed CUDA buffer with 128-byte rows; returns the m x n view."""
    import torch
    from . import _native
    dtype = torch.float64 if dtype is None else dtype
    es = 4 if dtype == torch.float32 else 8
    ld = -(-n * es // 128) * 128 // es
    return torch.zeros((m, ld), dtype=dtype, device=_native.device())[:, :n]


def _dev_normal(rng, m, n, loc=0.0, scale=1.0, rows=None):
    from . import _native
    A = _dev_matrix(m if rows is None else rows, n)
    _native.normal_fill(rng, A, m * n, loc, scale, ncol=n, rs=A.stride(0))
    return A


def _dmv(A, x, transpose=False):
    from . import _native
    return _native.dense_matvec(A, x, transpose).cpu().numpy()


def _dev_tall_lasso(m, n, seed, dtype=np.float64):
    import torch
    from . import _native
    r_a, r_v, r_n = _rngs("lasso", seed, 3)
    A = _dev_normal(r_a, m, n)
    v = _plant(r_v, n)
    b = _dmv(A, v) + r_n.normal(0.0, 0.5, size=m)
    lam = 0.2 * float(np.max(np.abs(_dmv(A, b, True))))
    if np.dtype(dtype) == np.float32:
        A32 = _dev_matrix(m, n, torch.float32)
        _native.convert_matrix(A, A32)
        A = A32
        b = b.astype(np.float32).astype(np.float64)
        lam = float(np.float32(lam))
    f = SeparableFunction.from_arrays(BaseFunction.SQUARE, size=m, b=b)
    g = SeparableFunction.from_arrays(BaseFunction.ABS, size=n, c=lam)
    return GraphFormProblem(A, f, g), {"v": v, "b": b, "lam": lam}


def _dev_generate(s):
    fam, m, n = s.family, s.m, s.n
    if fam == "lasso":
        _need(m < n, "lasso needs m < n")
        return _dev_tall_lasso(m, n, s.seed)
    if fam == "basis_pursuit":
        _need(m > n, "basis_pursuit needs m > n")
        r_a, r_v = _rngs(fam, s.seed, 2)
        A = _dev_normal(r_a, m, n)
        v = _plant(r_v, n)
        b = _dmv(A, v)
        f = SeparableFunction.from_arrays(BaseFunction.IND_EQ0, size=m, b=b)
        return GraphFormProblem(A, f, SeparableFunction.uniform(BaseFunction.ABS, n)), {"v": v, "b": b}
    if fam == "entropy_max":
        _need(m < n, "entropy_max needs m < n")
        r_a, r_v = _rngs(fam, s.seed, 2)
        A = _dev_normal(r_a, m, n, 0.0, np.sqrt(n), rows=m + 1)
        v = r_v.random(n)
        b = _dmv(A[:m], v) / v.sum()
        A[m].fill_(1.0)
        f = SeparableFunction.from_arrays([BaseFunction.IND_LE0] * m + [BaseFunction.IND_EQ0],
                                          b=np.concatenate([b, [1.0]]))
        return GraphFormProblem(A, f, SeparableFunction.uniform(BaseFunction.NEG_ENTR, n)), {"v": v, "b": b}
    if fam == "huber_fit":
        _need(m > n, "huber_fit needs m > n")
        r_a, r_v, r_e, r_o = _rngs(fam, s.seed, 4)
        A = _dev_normal(r_a, m, n, 0.0, np.sqrt(n))
        v = r_v.normal(0.0, 1.0 / np.sqrt(n), size=n)
        noise = r_e.normal(0.0, 0.5, size=m)
        out = r_o.random(m) >= 0.95
        noise[out] = r_o.random(out.sum()) * 10.0
        b = _dmv(A, v) + noise
        f = SeparableFunction.from_arrays(BaseFunction.HUBER, size=m, b=b)
        return (GraphFormProblem(A, f, SeparableFunction.uniform(BaseFunction.ZERO, n)),
                {"v": v, "b": b, "outlier_mask": out})
    if fam == "logistic":
        _need(m > n, "logistic needs m > n")
        r_a, r_v, r_l = _rngs(fam, s.seed, 3)
        A = _dev_normal(r_a, m, n)
        v = _plant(r_v, n)
        p0 = 1.0 / (1.0 + np.exp(-_dmv(A, v)))
        lab = np.where(r_l.random(m) < p0, 0.0, 1.0)
        lam = 0.1 * float(np.max(np.abs(_dmv(A, 0.5 - lab, True))))
        f = SeparableFunction.from_arrays(BaseFunction.LOGISTIC, size=m, d=-lab)
        g = SeparableFunction.from_arrays(BaseFunction.ABS, size=n, c=lam)
        return GraphFormProblem(A, f, g), {"v": v, "labels": lab, "lam": lam}
    if fam == "lp":
        _need(m > n, "lp needs m > n")
        r_a, r_v, r_e, r_u = _rngs(fam, s.seed, 4)
        A = _dev_normal(r_a, m, n)
        v = r_v.normal(0.0, 1.0 / np.sqrt(n), size=n)
        b = _dmv(A, v) + r_e.random(m) * 0.1
        u = r_u.random(m)
        c = -_dmv(A, u, True)
        f = SeparableFunction.from_arrays(BaseFunction.IND_LE0, size=m, b=b)
        g = SeparableFunction.from_arrays(BaseFunction.ZERO, size=n, d=c)
        return GraphFormProblem(A, f, g), {"v": v, "u": u, "b": b, "c": c}
    if fam == "nnls":
        _need(m > n, "nnls needs m > n")
        r_a, r_v, r_e = _rngs(fam, s.seed, 3)
        A = _dev_normal(r_a, m, n)
        v = r_v.normal(1.0 / n, 1.0 / np.sqrt(n), size=n)
        b = _dmv(A, v) + r_e.normal(0.0, 0.5, size=m)
        f = SeparableFunction.from_arrays(BaseFunction.SQUARE, size=m, b=b)
        return GraphFormProblem(A, f, SeparableFunction.uniform(BaseFunction.IND_GE0, n)), {"v": v, "b": b}
    if fam == "portfolio":
        from . import _native
        k = m
        _need(n > k, "portfolio needs n > k (pass the factor count as m)")
        r_f, r_d, r_mu = _rngs(fam, s.seed, 3)
        A = _dev_matrix(k + 1, n)
        _native.normal_fill(r_f, A, n * k, ncol=k, rs=1, cs=A.stride(0))   # F (n x k) written as F.T
        A[k].fill_(1.0)
        D = r_d.random(n) * np.sqrt(k)
        mu = r_mu.normal(size=n)
        f = SeparableFunction.from_arrays([BaseFunction.ZERO] * k + [BaseFunction.IND_EQ0],
                                          b=np.concatenate([np.zeros(k), [1.0]]),
                                          e=np.concatenate([np.full(k, 2.0), [0.0]]))
        g = SeparableFunction.from_arrays(BaseFunction.IND_GE0, size=n, d=-mu, e=2.0 * D)
        return GraphFormProblem(A, f, g), {"D": D, "mu": mu, "gamma_risk": 1.0}
    if fam == "svm":
        from . import _native
        _need(m > n, "svm needs m > n")
        (r_a,) = _rngs(fam, s.seed, 1)
        lab = np.where(np.arange(m) < m // 2, 1.0, -1.0)
        A = _dev_normal(r_a, m, n, 0.0, 1.0 / np.sqrt(n))
        _native.rows_affine(A, lab, lab / n)                                # lab * (A + lab / n)
        f = SeparableFunction.from_arrays(BaseFunction.MAX_POS0, size=m, b=-1.0, c=1.0)
        g = SeparableFunction.from_arrays(BaseFunction.ZERO, size=n, e=2.0)
        return GraphFormProblem(A, f, g), {"labels": lab, "lam": 1.0}
    raise ParameterError(f"unknown family {fam!r}")


def generate(spec: GenSpec, device: bool = False):
    """One instance of ``spec`` -> ``(problem, metadata)`` (generators.py:257-264).
    ``device=True`` draws the matrix on the GPU (same stream, same values)
    and returns it as a CUDA tensor."""
    problem, meta = (_dev_generate if device else _BUILD[spec.family])(spec)
    meta.update(family=spec.family, m=spec.m, n=spec.n, seed=spec.seed,
                rows=problem.m, cols=problem.n)
    return problem, meta

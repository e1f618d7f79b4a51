"""GPU: on-device input synthesis.

gf_normal_fill must reproduce numpy's Generator(PCG64).normal bit for bit --
the stream behind every reference generator -- so an instance drawn on the
device has exactly the reference's matrix (same SHA-256 as the host draw,
and as the fixtures made by the reference itself).  Vectors derived through
A @ v run in a different summation order than numpy's BLAS and are compared
to 1e-12.
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import _native, instances
from tests import _cases

pytestmark = pytest.mark.gpu


def _sha(A):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(A, np.float64)).tobytes()).hexdigest()


@pytest.mark.parametrize("seed,count,loc,scale", [(0, 1, 0.0, 1.0), (1, 7, 0.0, 1.0), (2, 1000, 0.5, 2.0),
                                                  (3, 1_000_003, 0.0, 1.0), (4, 3_000_000, -1.0, 0.25),
                                                  (6, 20_000_000, 0.0, 1.0)])
def test_normal_fill_is_numpy_bit_for_bit(seed, count, loc, scale):
    ref = np.random.default_rng(seed).normal(loc, scale, size=count)
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    _native.normal_fill(np.random.default_rng(seed), out, count, loc, scale)
    got = out.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: {got[bad[:5]]} vs {ref[bad[:5]]}"
    if count >= 1_000_000:   # the tail path (|z| > 3.654, log1p) was exercised
        assert np.sum(np.abs(ref - loc) > 3.6541528853610088 * scale) > 100


def test_normal_fill_fp32_and_strided_layouts():
    rng_seed, m, n = 11, 300, 77
    ref = np.random.default_rng(rng_seed).normal(size=(m, n))
    A = instances._dev_matrix(m, n, torch.float32)
    _native.normal_fill(np.random.default_rng(rng_seed), A, m * n, ncol=n, rs=A.stride(0))
    np.testing.assert_array_equal(A.cpu().numpy(), ref.astype(np.float32))
    # transposed placement (portfolio's F.T)
    T = instances._dev_matrix(n, m)
    _native.normal_fill(np.random.default_rng(rng_seed), T, m * n, ncol=n, rs=1, cs=T.stride(0))
    np.testing.assert_array_equal(T.cpu().numpy(), ref.T)


FAMILIES = [("lasso", 60, 200), ("basis_pursuit", 300, 80), ("entropy_max", 40, 150), ("huber_fit", 300, 60),
            ("logistic", 400, 50), ("lp", 300, 120), ("nnls", 300, 90), ("portfolio", 8, 120), ("svm", 400, 60)]


@pytest.mark.parametrize("family,m,n", FAMILIES)
def test_device_generate_matches_host(family, m, n):
    spec = instances.GenSpec(family, m, n, 5)
    hp, hm = instances.generate(spec)
    dp, dm = instances.generate(spec, device=True)
    assert _native.is_torch(dp.A) and dp.A.is_cuda
    A = dp.A.cpu().numpy()
    np.testing.assert_array_equal(A, np.asarray(hp.A))             # the matrix, bit for bit
    for part in ("f", "g"):
        hs, ds = getattr(hp, part), getattr(dp, part)
        np.testing.assert_array_equal(hs.h, ds.h)
        for k in "abcde":
            np.testing.assert_allclose(getattr(ds, k), getattr(hs, k), rtol=1e-12, atol=1e-12)
    for k in ("labels", "lam", "v", "u"):
        if k in hm:
            np.testing.assert_allclose(dm[k], hm[k], rtol=1e-12)


def test_device_tall_lasso_matches_reference_fixture():
    """The bench family: the device draw hashes to the SHA the reference's own
    fixture recorded (tests/golden/make_golden.py), fp64 and fp32 protocol."""
    fx = _cases.load("solve_lasso_tall_20000x500")
    prob, meta = instances.tall_lasso(20000, 500, 0, device=True)
    assert _sha(prob.A.cpu().numpy()) == str(fx["sha_A"])
    np.testing.assert_allclose(prob.f.b, fx["f_b"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(prob.g.c, fx["g_c"], rtol=1e-12)
    fx32 = _cases.load("solve_lasso_tall_20000x500_r32")
    p32, _ = instances.tall_lasso(20000, 500, 0, dtype=np.float32, device=True)
    assert p32.A.dtype == torch.float32
    assert _sha(p32.A.cpu().numpy()) == str(fx32["sha_A"])
    # and it solves like the host instance
    res = gf.solve(prob)
    assert res.status.value == str(fx["status"]) and res.iterations == int(fx["iterations"])

"""GPU side of the file loader (streamed straight to the device) and of the
equilibration diagnostics, against the reference's files and values."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import io as gio

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
IO = os.path.join(GOLDEN, "io")


def test_raw_matrix_streams_to_device_in_chunks(tmp_path, monkeypatch):
    A = np.random.default_rng(3).normal(size=(3001, 129))
    gio.write_raw_matrix(tmp_path / "a.bin", A)
    monkeypatch.setattr(gio, "_CHUNK_BYTES", 129 * 8 * 100)   # 31 chunks, both staging buffers cycle
    D = gio.read_raw_matrix(tmp_path / "a.bin", device=True)
    assert D.is_cuda and D.dtype == torch.float64 and D.stride(0) % 16 == 0
    np.testing.assert_array_equal(D.cpu().numpy(), A)
    D32 = gio.read_raw_matrix(tmp_path / "a.bin", device=True, dtype=np.float32)
    np.testing.assert_array_equal(D32.cpu().numpy(), A.astype(np.float32))


def test_device_problem_solves_like_host_problem():
    host = gio.load_problem(os.path.join(IO, "binref.json"))
    dev = gio.load_problem(os.path.join(IO, "binref.json"), device=True)
    assert dev.A.is_cuda
    np.testing.assert_array_equal(dev.A.cpu().numpy(), np.asarray(host.A))
    r1, r2 = gf.solve(host), gf.solve(dev)
    assert r1.iterations == r2.iterations and r1.status is r2.status
    np.testing.assert_array_equal(r1.x, r2.x)


def test_errors_are_the_reference_errors_on_the_device_path():
    exp = json.load(open(os.path.join(IO, "expected.json")))
    for name in ("bad_magic.bin", "short_header.bin", "wrong_size.bin"):
        with pytest.raises(gf.ProblemFormatError) as ei:
            gio.read_matrix(os.path.join(IO, name), device=True)
        assert "error: " + str(ei.value).replace(IO, "<dir>") == exp[name]


def test_equilibration_diagnostics_match_reference():
    ref = json.load(open(os.path.join(GOLDEN, "equil_diag.json")))
    z = np.load(os.path.join(GOLDEN, "equil.npz"))
    for key, want in ref.items():
        name, tag = key.split("|")
        A = z[f"{name}_A"]
        d, e = {"eq": (z[f"{name}_d"], z[f"{name}_e"]), "even": (z[f"{name}_rd"], z[f"{name}_re"]),
                "ones": (np.ones(A.shape[0]), np.ones(A.shape[1]))}[tag]
        rep = gf.check_equilibrated(A, d, e, tol=0.05).as_dict()
        for k in ("identity_abs", "identity_rel", "frobenius_ratio", "tol", "rows_ok", "cols_ok"):
            assert rep[k] == pytest.approx(want[k], rel=1e-10, abs=1e-14), (key, k)
        for k in ("row_deviation", "col_deviation"):
            assert rep[k] == pytest.approx(want[k], rel=1e-6, abs=1e-13), (key, k)
        obj = gf.equilibration_objective(A, d, e, float(z[f"{name}_gamma"]))
        assert obj == pytest.approx(want["objective"], rel=1e-12), key


def test_equilibrate_on_sweep_matches_reference():
    """on_sweep(k, d, e) after every sweep (equilibration.py:178-179)."""
    z = np.load(os.path.join(GOLDEN, "equil.npz"))
    sw = np.load(os.path.join(GOLDEN, "equil_sweeps.npz"))
    for name in ("gauss_300x120", "wide_80x200", "zero_row_60x30", "scaled_150x150"):
        rec = []
        eq = gf.equilibrate(z[f"{name}_A"], on_sweep=lambda k, d, e: rec.append((k, d, e)))
        assert [r[0] for r in rec] == list(sw[f"{name}_k"]) and eq.iterations == len(rec)
        for k, d, e in rec:
            np.testing.assert_allclose(d, sw[f"{name}_d{k}"], rtol=1e-12)
            np.testing.assert_allclose(e, sw[f"{name}_e{k}"], rtol=1e-12)
    with pytest.raises(ZeroDivisionError):   # the observer's exception reaches the caller
        gf.equilibrate(z["gauss_300x120_A"], on_sweep=lambda k, d, e: 1 / 0)

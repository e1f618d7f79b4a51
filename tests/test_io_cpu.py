"""Problem / matrix file formats against the reference's own files and
parses (tests/golden/io/, written by tests/golden/make_golden_io.py with the
reference's save_problem / write_raw_matrix, and read back by its loaders)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_1503_08366_b200 import io as gio
from paper_1503_08366_b200.errors import ProblemFormatError

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
EXPECTED = json.load(open(os.path.join(IO, "expected.json")))
PARSED = np.load(os.path.join(IO, "parsed.npz"))


def _load(name):
    path = os.path.join(IO, name)
    return gio.load_problem(path) if name.endswith(".json") else gio.read_matrix(path)


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_loaders_match_reference(name):
    exp = EXPECTED[name]
    if exp == "ok":
        got = _load(name)
        if name.endswith(".json"):
            np.testing.assert_array_equal(np.asarray(got.A), PARSED[name + ":A"])
            for part in ("f", "g"):
                for k in "habcde":
                    np.testing.assert_array_equal(np.asarray(getattr(getattr(got, part), k)),
                                                  PARSED[f"{name}:{part}_{k}"], err_msg=f"{part}.{k}")
        else:
            np.testing.assert_array_equal(got, PARSED[name])
    else:
        with pytest.raises(ProblemFormatError) as ei:
            _load(name)
        assert "error: " + str(ei.value).replace(IO, "<dir>") == exp


def test_writers_reproduce_reference_files(tmp_path):
    p = gio.load_problem(os.path.join(IO, "inline.json"))
    gio.save_problem(tmp_path / "inline.json", p)
    assert json.loads((tmp_path / "inline.json").read_text()) == json.loads(open(os.path.join(IO, "inline.json")).read())
    gio.save_problem(tmp_path / "binref.json", p, matrix_path="A.bin")
    assert json.loads((tmp_path / "binref.json").read_text()) == json.loads(open(os.path.join(IO, "binref.json")).read())
    assert (tmp_path / "A.bin").read_bytes() == open(os.path.join(IO, "A.bin"), "rb").read()
    gio.write_raw_matrix(tmp_path / "r.bin", PARSED["raw_7x3.bin"])
    assert (tmp_path / "r.bin").read_bytes() == open(os.path.join(IO, "raw_7x3.bin"), "rb").read()

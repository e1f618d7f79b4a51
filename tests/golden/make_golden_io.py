"""Golden files for the problem/matrix formats, written and read by the
REFERENCE (run where /root/reference exists):

    python tests/golden/make_golden_io.py

Writes tests/golden/io/: problem files saved by the reference's
save_problem (inline A, A in a raw .bin, A in a Matrix Market file), a raw
matrix from write_raw_matrix, malformed files, and expected.json /
parsed.npz with what the reference's loaders return (arrays, or the
ProblemFormatError message).
"""

from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import graphform as gf  # noqa: E402  (the reference)
from graphform import io as gio  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2024)
    m, n = 12, 5
    A = rng.normal(size=(m, n))
    kinds = list(gf.BaseFunction)
    f = gf.SeparableFunction.from_arrays([kinds[i % 10] for i in range(m)], a=rng.uniform(0.5, 2, m),
                                         b=rng.normal(size=m), c=np.where(np.arange(m) % 4 == 0, 1.0, 2.5),
                                         d=np.where(np.arange(m) % 3 == 0, 0.0, 0.25), e=np.zeros(m))
    g = gf.SeparableFunction.from_arrays(gf.BaseFunction.ABS, size=n, c=0.3)
    prob = gf.GraphFormProblem(A, f, g)
    gio.save_problem(os.path.join(OUT, "inline.json"), prob)
    gio.save_problem(os.path.join(OUT, "binref.json"), prob, matrix_path="A.bin")
    gio.save_problem(os.path.join(OUT, "mtxref.json"), prob, matrix_path="A.mtx")
    gio.write_raw_matrix(os.path.join(OUT, "raw_7x3.bin"), rng.normal(size=(7, 3)))
    # malformed inputs
    with open(os.path.join(OUT, "bad_magic.bin"), "wb") as fh:
        fh.write(struct.pack("<8sII", b"NOTAMATX", 2, 2) + np.zeros(4).tobytes())
    with open(os.path.join(OUT, "short_header.bin"), "wb") as fh:
        fh.write(b"GFMAT")
    with open(os.path.join(OUT, "wrong_size.bin"), "wb") as fh:
        fh.write(struct.pack("<8sII", b"GFMATRIX", 3, 3) + np.zeros(8).tobytes())
    with open(os.path.join(OUT, "bad.json"), "w") as fh:
        fh.write('{"m": 2, "n": 2,\n "A": [1, 2, 3,}')
    docs = {
        "missing_g.json": {"m": 1, "n": 1, "A": [[1.0]], "f": [{"h": "Square"}]},
        "term_count.json": {"m": 2, "n": 1, "A": [[1.0], [2.0]], "f": [{"h": "Square"}], "g": [{"h": "Abs"}]},
        "unknown_key.json": {"m": 1, "n": 1, "A": [[1.0]], "f": [{"h": "Square", "q": 1}], "g": [{"h": "Abs"}]},
        "bad_kind.json": {"m": 1, "n": 1, "A": [[1.0]], "f": [{"h": "Cube"}], "g": [{"h": "Abs"}]},
        "flat_size.json": {"m": 2, "n": 2, "A": [1.0, 2.0, 3.0], "f": [{"h": "Zero"}] * 2, "g": [{"h": "Zero"}] * 2},
        "flat_ok.json": {"m": 2, "n": 2, "A": [1.0, 2.0, 3.0, 4.0], "f": [{"h": "ind_le0", "b": 1}] * 2,
                         "g": [{"h": "IndGe0"}, {"h": "max-pos0", "e": 0.5}]},
        "neg_m.json": {"m": 0, "n": 1, "A": [], "f": [], "g": [{"h": "Abs"}]},
        "bad_param.json": {"m": 1, "n": 1, "A": [[1.0]], "f": [{"h": "Square", "a": "x"}], "g": [{"h": "Abs"}]},
        "shape_mismatch.json": {"m": 3, "n": 5, "A": "A.bin", "f": [{"h": "Zero"}] * 3, "g": [{"h": "Zero"}] * 5},
    }
    for name, doc in docs.items():
        with open(os.path.join(OUT, name), "w") as fh:
            json.dump(doc, fh)
    expected, arrays = {}, {}
    for name in sorted(os.listdir(OUT)):
        path = os.path.join(OUT, name)
        if name.endswith(".json") and name != "expected.json":
            try:
                p = gio.load_problem(path)
                A_ = p.A.toarray() if hasattr(p.A, "toarray") else np.asarray(p.A)
                arrays[name + ":A"] = A_
                for part in ("f", "g"):
                    for k in "habcde":
                        arrays[f"{name}:{part}_{k}"] = np.asarray(getattr(getattr(p, part), k))
                expected[name] = "ok"
            except gf.ProblemFormatError as exc:
                expected[name] = "error: " + str(exc).replace(OUT, "<dir>")
        elif name.endswith(".bin") or name.endswith(".mtx"):
            try:
                arrays[name] = np.asarray(gio.read_matrix(path))
                expected[name] = "ok"
            except gf.ProblemFormatError as exc:
                expected[name] = "error: " + str(exc).replace(OUT, "<dir>")
    with open(os.path.join(OUT, "expected.json"), "w") as fh:
        json.dump(expected, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "parsed.npz"), **arrays)
    print(json.dumps(expected, indent=1))


if __name__ == "__main__":
    main()

"""Benchmark sweep harness against the reference's
``graphform bench``: the dimension rule on a grid (CPU) and a whole small
sweep's CSVs (GPU) -- same records, iteration counts and statuses, objectives
to 1e-6 (tests/golden/make_golden_bench.py ran the reference)."""

from __future__ import annotations

import csv
import json
import os

import pytest

from paper_1503_08366_b200 import sweep

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_bench_dims_match_reference():
    ref = json.load(open(os.path.join(GOLDEN, "bench_dims.json")))
    for key, want in ref.items():
        fam, nnz, asp = key.split("|")
        num, _, den = asp.partition(":")
        got = sweep.bench_dims(fam, float(nnz), float(num) / float(den))
        assert (list(got) if got else None) == want, key


def test_bench_fields_are_the_reference_schema():
    with open(os.path.join(GOLDEN, "bench_ref.csv")) as fh:
        assert tuple(next(csv.reader(fh))) == sweep.BENCH_FIELDS


@pytest.mark.gpu
def test_sweep_matches_reference_csv(tmp_path):
    spec = json.load(open(os.path.join(GOLDEN, "bench_ref_sweep.json")))
    recs, out, agg = sweep.run_bench(out=tmp_path / "b.csv", **spec)
    with open(os.path.join(GOLDEN, "bench_ref.csv")) as fh:
        ref = list(csv.DictReader(fh))
    with open(out) as fh:
        got = list(csv.DictReader(fh))
    assert len(got) == len(ref) == len(recs)
    for g, r in zip(got, ref):
        for k in ("family", "m", "n", "nnz", "iterations", "status"):
            assert g[k] == r[k], (k, g, r)
        assert float(g["objective"]) == pytest.approx(float(r["objective"]), rel=1e-6, abs=1e-9)
    with open(agg) as fh:
        rows = list(csv.reader(fh))
    with open(os.path.join(GOLDEN, "bench_ref_agg.csv")) as fh:
        ref_rows = list(csv.reader(fh))
    assert rows[0] == ref_rows[0]
    assert [r[:2] + r[3:] for r in rows[1:]] == [r[:2] + r[3:] for r in ref_rows[1:]]

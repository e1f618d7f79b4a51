"""Golden output of the REFERENCE's benchmark sweep (``graphform bench``,
cli.py:221-308) and of its dimension rule, for tests/test_sweep_*.py:

    python tests/golden/make_golden_bench.py

bench_ref.csv / bench_ref_agg.csv: the reference's CSVs for a small sweep;
bench_dims.json: _bench_dims over a grid of families x nnz x aspects.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from graphform import cli  # noqa: E402  (the reference)
from graphform.generators import FAMILIES  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SWEEP = dict(families="lasso,svm,nnls,huber_fit", nnz="1e4,4e4", aspects="4:1,1:4", seeds="0,1")


def main():
    dims = {}
    for fam in FAMILIES:
        for nnz in (1e2, 1e4, 3.3e5, 1e9):
            for asp in ("4:1", "1:4", "1:1", "10:1", "1:3"):
                num, _, den = asp.partition(":")
                d = cli._bench_dims(fam, nnz, float(num) / float(den))
                dims[f"{fam}|{nnz:g}|{asp}"] = list(d) if d else None
    with open(os.path.join(HERE, "bench_dims.json"), "w") as fh:
        json.dump(dims, fh, indent=0, sort_keys=True)
    args = argparse.Namespace(
        families=SWEEP["families"], nnz=SWEEP["nnz"], aspects=SWEEP["aspects"], seeds=SWEEP["seeds"],
        jobs=1, max_elements=5e7, out=os.path.join(HERE, "bench_ref.csv"), agg_out=None,
        rho=1.0, abs_tol=1e-4, rel_tol=1e-3, max_iter=10000, alpha=1.7, no_adaptive_rho=False,
        no_equil=False, indirect=False, gap_stop=False, verbose=False)
    cli._cmd_bench(args)
    with open(os.path.join(HERE, "bench_ref_sweep.json"), "w") as fh:
        json.dump(SWEEP, fh)


if __name__ == "__main__":
    main()

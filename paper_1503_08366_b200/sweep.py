"""Benchmark sweep over generated instances with the reference's CSV schema
(reference ``cli.py:31-34``, ``:183-308``).

``run_bench`` reproduces the reference's ``graphform bench`` sweep -- the
paper's time-vs-size study (Fig. 1): for each family, target element count
and row:col aspect that the family permits, the instance of each seed is
generated, solved, and recorded with the reference's ``BENCH_FIELDS``; an
aggregate CSV holds the mean solve time per (family, nnz).  Differences from
the reference, which runs the same sweep through a process pool on the CPU:
instances are drawn on the GPU by default (bit-identical matrices,
``instances.generate(..., device=True)``) and solved one after another on the
current device; the element budget defaults to 2e9 instead of 5e7 (a B200
holds and solves 1e9-entry instances in well under a second).
"""

from __future__ import annotations

import csv
from pathlib import Path

import numpy as np

from .errors import GraphFormError, ParameterError
from .instances import FAMILIES, GenSpec, canonical_family, generate
from .solver import SolverSettings, solve

__all__ = ["BENCH_FIELDS", "bench_dims", "bench_one", "run_bench"]

BENCH_FIELDS = (
    "family", "m", "n", "nnz", "iterations", "status",
    "solve_time_s", "setup_time_s", "objective", "r_pri", "r_dual",
)


def bench_dims(family: str, nnz: float, ratio: float):
    """Dimensions with ~nnz entries and row:col ratio for one family, or None
    when the family does not permit the orientation (cli.py:183-199)."""
    n = max(1, round(np.sqrt(nnz / ratio)))
    m = max(1, round(ratio * n))
    if family in ("entropy_max", "lasso"):
        if m >= n:
            return None
        m = max(1, m - 1)  # the stacked row keeps the emitted nnz near target
        return m, n
    if family == "portfolio":
        if m >= n:
            return None
        return max(1, m - 1), n
    if m <= n:
        return None
    return m, n


def bench_one(family, m, n, seed, settings_kwargs, device: bool = True) -> dict:
    """One generated instance, solved; a BENCH_FIELDS record (cli.py:202-218)."""
    problem, _ = generate(GenSpec(family=family, m=m, n=n, seed=seed), device=device)
    result = solve(problem, SolverSettings(**settings_kwargs))
    return {
        "family": family,
        "m": problem.m,
        "n": problem.n,
        "nnz": problem.m * problem.n,
        "iterations": result.iterations,
        "status": result.status.value,
        "solve_time_s": f"{result.solve_time:.6f}",
        "setup_time_s": f"{result.setup_time:.6f}",
        "objective": f"{result.objective:.12g}",
        "r_pri": f"{result.primal_residual:.6g}",
        "r_dual": f"{result.dual_residual:.6g}",
    }


def _parse_list(text, conv, what):
    try:
        return [conv(x) for x in str(text).split(",") if x.strip()]
    except ValueError as exc:
        raise ParameterError(f"bad {what} list {text!r}: {exc}") from exc


def run_bench(families="all", nnz="1e2,1e4", aspects="4:1,1:4", seeds="0,1,2", out="bench.csv",
              agg_out=None, max_elements: float = 2e9, device: bool = True, rho=1.0, abs_tol=1e-4,
              rel_tol=1e-3, max_iter=10000, alpha=1.7, adaptive_rho=True, equilibrate=True,
              projection="direct"):
    """The reference's bench sweep (cli.py:221-308): writes ``out`` (one
    record per instance, sorted like the reference) and the aggregate CSV
    (default ``<out stem>_agg<suffix>``).  Returns (records, out, agg_out)."""
    if str(families).strip().lower() == "all":
        fams = list(FAMILIES)
    else:
        try:
            fams = [canonical_family(f) for f in str(families).split(",") if f.strip()]
        except GraphFormError:
            raise
    if not fams:
        raise ParameterError("empty family list")
    nnz_list = _parse_list(nnz, float, "nnz")
    seed_list = _parse_list(seeds, int, "seed")
    ratios = []
    for token in str(aspects).split(","):
        num, _, den = token.partition(":")
        try:
            ratios.append(float(num) / float(den or "1"))
        except ValueError as exc:
            raise ParameterError(f"bad aspect {token!r}") from exc
    jobs = []
    for family in fams:
        for target in nnz_list:
            if target > max_elements:
                raise ParameterError(f"nnz {target:g} exceeds max_elements {max_elements:g}")
            for ratio in ratios:
                dims = bench_dims(family, target, ratio)
                if dims is None:
                    continue
                for seed in seed_list:
                    jobs.append((family, *dims, seed, target))
    settings_kwargs = dict(rho0=rho, abs_tol=abs_tol, rel_tol=rel_tol, max_iter=max_iter, alpha=alpha,
                           adaptive_rho=adaptive_rho, equilibrate=equilibrate, projection=projection)
    records = []
    for fam, m, n, seed, target in jobs:
        rec = bench_one(fam, m, n, seed, settings_kwargs, device=device)
        rec["_target"] = target
        records.append(rec)
    records.sort(key=lambda r: (r["family"], r["_target"], r["m"], r["nnz"]))
    out = Path(out)
    with open(out, "w", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=BENCH_FIELDS, extrasaction="ignore")
        writer.writeheader()
        writer.writerows(records)
    agg_path = Path(agg_out) if agg_out else out.with_name(out.stem + "_agg" + out.suffix)
    groups = {}
    for rec in records:
        groups.setdefault((rec["family"], rec["_target"]), []).append(float(rec["solve_time_s"]))
    with open(agg_path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["family", "nnz", "mean_solve_time_s", "runs"])
        for (family, target), times in sorted(groups.items()):
            writer.writerow([family, f"{target:g}", f"{float(np.mean(times)):.6f}", len(times)])
    return records, out, agg_path

"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel counts / totals / shares, split into setup (before the first
fused/row pass) and iterations."""
import collections
import csv
import re
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) == 15 and r[0] != "ID"]
launches = [(re.sub(r"\(.*", "", r[4]).replace("void ", ""), float(r[14]) / 1e3) for r in rows]
names = [n for n, _ in launches]
first = next(i for i, n in enumerate(names)
             if "fused_rowcol" in n or re.search(r"rowgemv_kernel<\w+, 2", n))
# the setup preceding the first iteration: walk back to the first equilibration launch of that prepare
setup_start = max(i for i, n in enumerate(names[:first]) if "sq_row" in n or "equil" in n.lower()) if first else 0
while setup_start > 0 and ("sq_row" in names[setup_start - 1] or "col_update" in names[setup_start - 1]
                           or "sum_parts" in names[setup_start - 1]):
    setup_start -= 1


def table(seg, title):
    tot = sum(t for _, t in seg)
    agg = collections.OrderedDict()
    for n, t in seg:
        c, s = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, s + t)
    print(f"== {title}: {len(seg)} launches, {tot / 1e3:.3f} ms device time (serialised, cold cache)")
    print(f"{'kernel':60s} {'count':>6s} {'total_ms':>10s} {'avg_us':>10s} {'share':>7s}")
    for n, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:60]:60s} {c:6d} {s / 1e3:10.3f} {s / c:10.2f} {100 * s / tot:6.1f}%")
    print()


print(f"# {path}: {len(launches)} launches captured")
table(launches[:first], "setup + earlier calls (equilibration, Gram, Cholesky, TRTRI, inverse)")
table(launches[first:], "ADMM iterations (warm-up + timed + profiled pass)")

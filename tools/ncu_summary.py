"""Summarise an ncu report: key raw metrics + hottest SASS lines by stall samples."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        print(f"{k:60s} {vals[i]} {units[i]}")
stalls = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            stalls.append((float(vals[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
print("stall samples:", ", ".join(f"{n}={int(v)}" for v, n in sorted(stalls, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = None
data = []
for r in srows:
    if "Warp Stall Sampling (All Samples)" in r:
        h = r
        continue
    if h and len(r) == len(h):
        try:
            data.append((int(r[h.index("Warp Stall Sampling (All Samples)")]), r[h.index("Source")], r[h.index("Address")]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}")
for s, line, addr in sorted(data, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {addr} {line.strip()[:90]}")

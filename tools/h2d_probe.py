"""Dev probe: host->device copy rates for the 4 GB C5 matrix from pinned memory:
one 1-D copy, one 2-D pitched copy (20000 B rows -> 20096 B device rows, what
gf_matrix_create does), the same split over 2 and 4 streams."""
import time
import torch
m, n, ldd = 200000, 5000, 5024
h = torch.empty(m * n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(m * ldd, dtype=torch.float32, device="cuda")
dv = d.view(m, ldd)[:, :n]
hv = h.view(m, n)
def timeit(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best
gb = m * n * 4 / 1e9
t = timeit(lambda: d[: m * n].copy_(h, non_blocking=True)); print(f"1-D   {t*1e3:.1f} ms {gb/t:.1f} GB/s")
t = timeit(lambda: dv.copy_(hv, non_blocking=True)); print(f"2-D   {t*1e3:.1f} ms {gb/t:.1f} GB/s")
for ns in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    def split():
        for i, s in enumerate(streams):
            r0, r1 = m * i // ns, m * (i + 1) // ns
            with torch.cuda.stream(s):
                dv[r0:r1].copy_(hv[r0:r1], non_blocking=True)
    t = timeit(split); print(f"2-D x{ns} streams {t*1e3:.1f} ms {gb/t:.1f} GB/s")

"""Benchmark: ADMM iterations/s on dense Lasso (BASELINE.json metric).

Workload (BASELINE.json configs[4], the paper's billion-coefficient scale):
dense Lasso 200000 x 5000 (1e9 coefficients), A ~ N(0,1) rounded to fp32,
f = Square(b), g = lambda*Abs, built by the reference's Lasso recipe
(instances.tall_lasso, bit-identical streams) on the host -- synthetic data.
A is 4 GB in fp32, far larger than the 126 MB L2, so every timed iteration
streams it from HBM (no L2 flush needed).

A "step" is one ADMM iteration (solver.py:329-428) of that solve.
  value  iterations/s with A resident in HBM: W warm-up iterations, then K
         iterations timed with CUDA events on the solver's stream (barrier +
         synchronize on both sides, max over ranks).
  e2e    the same metric through the public API from HOST buffers: a full
         ``solve(problem)`` on a pinned host copy of A -- H2D of A and the term
         arrays, equilibration, Gram + Cholesky, iterations to eps_rel = 1e-3
         and the D2H of x, y, mu, nu -- iterations / wall time.  Its wall time
         is also reported as time_to_eps_s.
  roofline  for the dominant kernel (row pass over A_hat), algorithmic bytes
         m*n*4 per launch / its CUDA-event duration, against the measured HBM
         copy peak (MEASURED_PEAKS.json).
  cpu_baseline  the CPU oracle port (oracle/graphform_oracle.py, fp64 numpy
         with all host threads) timed on a bounded row sample of the same
         instance; iterations/s scaled to the full row count.

--impl reference runs the CPU oracle port (the reference is pure Python and
cannot travel to the GPU box) on the same full-size instance: prepare, then
W + K iterations, timing the K.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_FULL, N_FULL = 200_000, 5_000
METRIC = "admm_iters_per_s"


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def ncu_traffic(kernel, m, n):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel``
    from the committed ``ncu --set full`` capture (profiles/traffic.json),
    when it was taken on this exact per-rank shape; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)[kernel]
    except (OSError, KeyError, ValueError):
        return None
    return d["dram_bytes_per_launch"] if (d.get("m"), d.get("n")) == (m, n) else None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    fallback = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    try:
        with open(p) as f:
            d = json.load(f)
        if float(d.get("hbm_gbs", 0)) > 0:
            return d, "measured"
    except (OSError, ValueError, TypeError, AttributeError):
        pass
    return fallback, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        # NVML (the library behind nvidia-smi), initialised before the timed
        # region starts so that polling covers all of it
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            return N, h, mx
        except Exception:
            return None

    def _run(self):
        # NVML polled every 5 ms; falls back to the nvidia-smi CLI when pynvml
        # is unavailable
        if self._nv is not None:
            N, h, mx = self._nv
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.005)
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._nv = self._nvml()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def build_instance(m, n, rank=0, world=1):
    from paper_1503_08366_b200 import instances
    prob, meta = instances.tall_lasso(m, n, seed=0, dtype=np.float32)
    return prob, meta


def cpu_baseline(prob, sample_rows, iters=10):
    """Oracle port on the first `sample_rows` rows: iterations/s scaled to m."""
    from oracle import graphform_oracle as orc
    m = prob.m
    A = np.asarray(prob.A[:sample_rows], dtype=np.float64)
    f = orc.Terms(*(np.asarray(getattr(prob.f, k))[:sample_rows] for k in "habcde"))
    g = orc.Terms.of(prob.g)
    st = dict(abs_tol=1e-12, rel_tol=1e-12, max_iter=iters + 2)
    setup = orc.prepare(A, st)
    stamps = []
    orc.solve(A, f, g, st, setup=setup, callback=lambda *a: stamps.append(time.perf_counter()))
    dt = stamps[-1] - stamps[1]
    per_it = dt / (len(stamps) - 2)
    return {"value": (1.0 / per_it) * (sample_rows / m), "unit": "iters/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"first {sample_rows} of {m} rows ({sample_rows}x{prob.n} fp64), "
                      f"{len(stamps) - 2} timed iterations after prepare; iters/s scaled by {sample_rows}/{m}"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from oracle import graphform_oracle as orc
    m, n = args.m, args.n
    prob, _ = build_instance(m, n)
    A = np.asarray(prob.A, dtype=np.float64)
    f, g = orc.Terms.of(prob.f), orc.Terms.of(prob.g)
    # bounded sample: at most 20 timed iterations after at most 3 warm-up ones
    # (one CPU iteration of the full instance is ~1 s), so the arm finishes in
    # about a minute whatever --steps the driver passes
    k = max(1, min(args.steps, 20))
    w = max(1, min(args.warmup, 3))
    st = dict(abs_tol=1e-12, rel_tol=1e-12, max_iter=w + k)
    t0 = time.perf_counter()
    setup = orc.prepare(A, st)
    t_setup = time.perf_counter() - t0
    stamps = []
    orc.solve(A, f, g, st, setup=setup, callback=lambda *a: stamps.append(time.perf_counter()))
    dt = stamps[w + k - 1] - stamps[w - 1]
    val = k / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "iters/s", "n_gpus": world,
            "steps": k, "warmup": w, "ms_per_step": 1e3 * dt / k, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"dense Lasso {m}x{n} (tall_lasso seed 0, A rounded to fp32, fp64 arithmetic)",
                       "m": m, "n": n, "parallelism": "cpu"},
            "cpu_baseline": {"value": val, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"full instance; prepare {t_setup:.1f}s excluded; {k} iterations "
                                       f"after {w} warm-up (bounded: requested --steps {args.steps} "
                                       f"--warmup {args.warmup})"},
            "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import paper_1503_08366_b200 as gf
    from paper_1503_08366_b200 import _native, distributed, solver as slv
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    use_comm = world > 1 or args.force_comm
    if use_comm:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
        comm = distributed.init_comm()

    def sync():
        torch.cuda.synchronize()
        if use_comm:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if use_comm:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    m, n = args.m, args.n
    r0, r1 = distributed.row_range(m, rank, world)
    t_gen = time.perf_counter()
    full, meta = build_instance(m, n)
    host_generate_s = time.perf_counter() - t_gen
    # this rank's rows (row partition); the host copy of the
    # full matrix is dropped before any device work
    prob = gf.GraphFormProblem(np.ascontiguousarray(full.A[r0:r1]), full.f.slice(r0, r1), full.g)
    del full
    m_loc = r1 - r0
    peaks, peaks_kind = measured_peaks()
    # ---------------- e2e: full solve from pinned host memory ----------------
    e2e = None
    if not args.skip_e2e:
        A_pin = torch.from_numpy(prob.A).pin_memory()
        prob_pin = gf.GraphFormProblem(A_pin, prob.f, prob.g)
        e2e_runs = []
        for _ in range(5):   # the first call warms module load / allocator; best of the rest
            sync()
            t0 = time.perf_counter()
            res = gf.solve(prob_pin, comm=comm)
            torch.cuda.synchronize()
            e2e_runs.append((max_over_ranks([time.perf_counter() - t0])[0], res))
        e2e_time, res = min(e2e_runs[1:], key=lambda r: r[0]) if len(e2e_runs) > 1 else e2e_runs[-1]
        # phase breakdown of the same public-API path (diagnostic, not the headline)
        sync()
        t0 = time.perf_counter()
        setup_b = gf.prepare(prob_pin, comm=comm)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        run_b = slv._Run(setup_b, prob.f, prob.g, gf.SolverSettings(), None, None, m_loc)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        run_b.run(0)
        t3 = time.perf_counter()
        run_b.result()
        t4 = time.perf_counter()
        phases = {"prepare_s": t1 - t0, "solver_create_s": t2 - t1, "iterate_s": t3 - t2, "result_s": t4 - t3,
                  "iterations": int(run_b.state.iterations)}
        del run_b, setup_b
        h2d = prob.A.nbytes + sum(getattr(prob.f, k).nbytes for k in "abcde") + m_loc \
            + sum(getattr(prob.g, k).nbytes for k in "abcde") + n
        d2h = 8 * (2 * m_loc + 2 * n)
        e2e = {"value": res.iterations / e2e_time, "unit": "iters/s",
               "h2d_bytes_per_step": int(h2d / max(res.iterations, 1)),
               "d2h_bytes_per_step": int(d2h / max(res.iterations, 1)),
               "time_to_eps_s": e2e_time, "iterations": res.iterations, "status": res.status.value,
               "objective": res.objective, "setup_s": res.setup_time, "h2d_bytes_total": int(h2d),
               "runs_s": [round(r[0], 4) for r in e2e_runs], "phases": phases,
               "host_generate_s": host_generate_s}
        if world == 1:
            # the same instance drawn on the GPU (bit-identical
            # A from the reference's PCG64 stream) and solved -- time to eps with
            # no host generation and no 4 GB H2D copy
            from paper_1503_08366_b200 import instances
            sync()
            t0 = time.perf_counter()
            pdev, _ = instances.tall_lasso(m, n, 0, dtype=np.float32, device=True)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            rdev = gf.solve(pdev)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            same = bool(torch.equal(pdev.A, torch.from_numpy(prob.A).to(dev)))
            e2e["device_generated"] = {"generate_s": t1 - t0, "solve_s": t2 - t1, "time_to_eps_s": t2 - t0,
                                       "iterations": rdev.iterations, "status": rdev.status.value,
                                       "A_identical_to_host_draw": same}
            del pdev, rdev
    # ---------------- device-resident iteration timing ----------------
    setup = gf.prepare(prob, comm=comm)
    tight = gf.SolverSettings(abs_tol=1e-12, rel_tol=1e-12, max_iter=args.warmup + 2 * args.steps + 8)
    run = slv._Run(setup, prob.f, prob.g, tight, None, None, m_loc)
    run.run(args.warmup)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    L = _native.lib()
    import ctypes as C
    l0 = C.c_int64()
    _native.check(L.gf_solver_stats(run.handle, C.byref(l0), None, None))
    with ClockSampler(local) as clk:
        sync()
        e0.record(stream)
        st = run.run(args.steps)
        e1.record(stream)
        sync()
    ms = max_over_ranks([e0.elapsed_time(e1)])[0]
    l1 = C.c_int64()
    _native.check(L.gf_solver_stats(run.handle, C.byref(l1), None, None))
    assert st.status == 0 and st.k + 1 == args.warmup + args.steps, (st.status, st.k)
    value = args.steps / (ms / 1e3)
    # ---------------- per-kernel durations (profiled pass) ----------------
    _native.check(L.gf_solver_profile(run.handle, 1))
    run.run(args.steps)
    kms = (C.c_double * 8)()
    kcnt = (C.c_int64 * 8)()
    _native.check(L.gf_solver_stats(run.handle, None, kms, kcnt))
    names = ["ginv_gemv_xside", "row_pass_yside", "col_pass", "slab_reduce", "y_scalars", "zstep_controller",
             "allreduce", "fused_rowcol_yside"]
    kernels = {names[i]: {"avg_ms": kms[i] / kcnt[i], "count": int(kcnt[i])} for i in range(8) if kcnt[i]}
    es = 4 if setup.dtype == _native.GF_F32 else 8
    # dominant kernel: the pass over this rank's rows of A_hat (fused single
    # pass, or the row pass of the two-pass fallback); algorithmic bytes =
    # m_loc*n*s per launch
    dom = "fused_rowcol_yside" if "fused_rowcol_yside" in kernels else "row_pass_yside"
    alg_bytes = m_loc * n * es
    t_row = max_over_ranks([kernels[dom]["avg_ms"]])[0] / 1e3
    achieved = alg_bytes / t_row / 1e9
    peak = peaks["hbm_gbs"]
    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if es == 4 else "f64",
        "data": "synthetic (reference Lasso recipe, seed 0, A rounded to fp32)",
        "config": {"workload": f"dense Lasso {m}x{n} fp32 (BASELINE configs[4], 1e9 coefficients)",
                   "m": m, "n": n, "parallelism": f"row partition x{world}" + (" (NCCL all-reduce)" if use_comm else ""),
                   "rows_per_rank": m_loc,
                   "l2": "A is 4 GB >> 126 MB L2; no flush needed"},
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(dom, m_loc, n), "kernel": dom,
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_kind": peaks_kind,
                     # context: the kernel only reads A_hat; a bare TMA read ring on
                     # this part reaches ~7.34 TB/s (profiles/r01_readbw_probe.txt)
                     "read_stream_ceiling_gbs": 7344.0, "frac_of_read_ceiling": achieved / 7344.0},
        "kernels": kernels,
        "gpu_launches": int(l1.value - l0.value),
        "clocks": clk.summary(),
    }
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_baseline(prob, max(1, m // 10), iters=10)
    if rank == 0:
        print(json.dumps(line))
    del run, setup
    if use_comm:
        del comm
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=M_FULL)
    ap.add_argument("--n", type=int, default=N_FULL)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true",
                    help="profiling runs only: skip the end-to-end solves (the line then has e2e null)")
    ap.add_argument("--force-comm", action="store_true",
                    help="use the NCCL row-partition path even on one GPU (checks the multi-GPU plumbing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

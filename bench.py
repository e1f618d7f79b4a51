"""Benchmark: ADMM iterations/s on dense Lasso (BASELINE.json metric).

Workload (BASELINE.json configs[4], the paper's billion-coefficient scale):
dense Lasso 200000 x 5000 (1e9 coefficients), A ~ N(0,1) rounded to fp32,
f = Square(b), g = lambda*Abs, built by the reference's Lasso recipe drawn on
the GPU (instances.tall_lasso(device=True): bit-identical to the reference's
numpy streams) -- synthetic data.  A is 4 GB in fp32, far larger than the
126 MB L2, so every timed iteration streams it from HBM (no L2 flush needed).

A "step" is one ADMM iteration (solver.py:329-428) of that solve.
  value  iterations/s with A resident in HBM, fp32 matrix passes (configs[4]):
         W warm-up iterations, then K iterations timed with CUDA events on
         the solver's stream (barrier + synchronize on both sides, max over
         ranks).
  e2e    the same metric through the public API from HOST buffers: a full
         ``solve(problem)`` on a pinned host copy of A -- H2D of A and the term
         arrays, equilibration, Gram + Cholesky, iterations to eps_rel = 1e-3
         and the D2H of x, y, mu, nu -- iterations / wall time (best of runs
         2..5; the first run is reported as first_solve_s).
  roofline  for the dominant kernel (the fused pass over A_hat), algorithmic
         bytes m*n*s per launch / its CUDA-event duration, against the
         measured HBM copy peak (MEASURED_PEAKS.json).
  fp64   the same instance at the reference's own precision (fp64 matrix
         passes, what ``solve`` does by default): value, roofline and e2e.
  cpu_baseline  the CPU oracle port (oracle/graphform_oracle.py, fp64 numpy
         with all host threads) on the FULL instance, 5 iterations after 2
         warm-up -- the same code as the reference arm.

--gpus N without torchrun re-executes itself as N ranks (torchrun on
127.0.0.1); under torchrun WORLD_SIZE must equal --gpus.  Each rank draws the
instance on its GPU and keeps its row block (row partition, strong scaling).

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


def device_instance(m, n, rank, world):
    """This rank's rows of the bench instance, drawn on the GPU (the reference
    Lasso recipe: bit-identical to the host numpy streams, tests/
    test_gpu_generate.py) and rounded to fp32: rank r keeps rows
    row_range(m, r, world) -- no host draw, no 4 GB host copy per rank."""
    import paper_1503_08366_b200 as gf
    from paper_1503_08366_b200 import distributed, instances
    t0 = time.perf_counter()
    full, meta = instances.tall_lasso(m, n, seed=0, dtype=np.float32, device=True)
    r0, r1 = distributed.row_range(m, rank, world)
    A = full.A[r0:r1].clone() if world > 1 else full.A
    prob = gf.GraphFormProblem(A, full.f.slice(r0, r1), full.g)
    del full
    return prob, time.perf_counter() - t0


def host_instance(m, n):
    """The bench instance drawn on the host by the reference recipe
    (reference arm: nothing of this repo's CUDA path is used)."""
    from paper_1503_08366_b200 import instances
    prob, _ = instances.tall_lasso(m, n, seed=0, dtype=np.float32)
    return prob


def time_port(A, f, g, k, w):
    """The CPU oracle port (oracle/graphform_oracle.py: numpy fp64, all host
    threads through BLAS) on the full instance: prepare, then w + k
    iterations; returns (iterations/s over the last k, prepare seconds).  The
    same code times the reference arm and the cpu_baseline."""
    from oracle import graphform_oracle as orc
    A = np.asarray(A, dtype=np.float64)
    st = dict(abs_tol=1e-12, rel_tol=1e-12, max_iter=w + k)
    t0 = time.perf_counter()
    setup = orc.prepare(A, st)
    t_setup = time.perf_counter() - t0
    stamps = []
    orc.solve(A, orc.Terms.of(f), orc.Terms.of(g), st, setup=setup,
              callback=lambda *a: stamps.append(time.perf_counter()))
    dt = stamps[w + k - 1] - stamps[w - 1]
    return k / dt, t_setup


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    m, n = args.m, args.n
    prob = host_instance(m, n)
    # bounded sample: at most 20 timed iterations after at most 3 warm-up ones
    # (one CPU iteration of the full instance is ~0.3 s on 16 cores), so the
    # arm finishes in about a minute whatever --steps the driver passes
    k = max(1, min(args.steps, 20))
    w = max(1, min(args.warmup, 3))
    val, t_setup = time_port(prob.A, prob.f, prob.g, k, w)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "iters/s", "n_gpus": world,
            "steps": k, "warmup": w, "ms_per_step": 1e3 / val, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"dense Lasso {m}x{n} (tall_lasso seed 0, A rounded to fp32, fp64 arithmetic)",
                       "m": m, "n": n, "parallelism": "cpu"},
            "cpu_baseline": {"value": val, "unit": "iters/s", "cores": host_cores(), "kind": "port",
                             "sample": f"full instance; prepare {t_setup:.1f}s excluded; {k} iterations "
                                       f"after {w} warm-up (bounded: requested --steps {args.steps} "
                                       f"--warmup {args.warmup})"},
            "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


class Ctx:
    """Per-rank plumbing: device, optional NCCL communicator, barrier-synced
    timing and max-over-ranks reductions."""

    def __init__(self, args):
        import torch
        from paper_1503_08366_b200 import distributed
        self.torch = torch
        self.rank, self.world, self.local = env_rank()
        if args.gpus != self.world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={self.world}")
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.use_comm = self.world > 1 or args.force_comm
        self.comm = None
        if self.use_comm:
            import torch.distributed as dist
            self.dist = dist
            if self.world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl", device_id=self.dev)
            self.comm = distributed.init_comm()

    def sync(self):
        self.torch.cuda.synchronize()
        if self.use_comm:
            self.dist.barrier()
            self.torch.cuda.synchronize()

    def max_over_ranks(self, vals):
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self.dev)
        if self.use_comm:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def close(self):
        if self.use_comm:
            del self.comm
            self.dist.destroy_process_group()


KERNEL_NAMES = ["ginv_gemv_xside", "row_pass_yside", "col_pass", "slab_reduce", "y_scalars", "zstep_controller",
                "allreduce", "fused_rowcol_yside"]


def iteration_timing(cx, prob, settings, steps, warmup, peaks):
    """`value`: `steps` ADMM iterations with A_hat resident (after `warmup`),
    CUDA events on the solver's stream, barrier + synchronize on both sides,
    max over ranks; then a profiled pass of the same length for the per-kernel
    durations the roofline uses."""
    import ctypes as C
    import paper_1503_08366_b200 as gf
    from paper_1503_08366_b200 import _native, solver as slv
    torch = cx.torch
    m_loc, n = prob.m, prob.n
    setup = gf.prepare(prob, settings, comm=cx.comm)
    tight = gf.SolverSettings(abs_tol=1e-12, rel_tol=1e-12, max_iter=warmup + 2 * steps + 8,
                              precision=settings.precision)
    run = slv._Run(setup, prob.f, prob.g, tight, None, None, m_loc)
    run.run(warmup)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    L = _native.lib()
    l0, l1 = C.c_int64(), C.c_int64()
    _native.check(L.gf_solver_stats(run.handle, C.byref(l0), None, None))
    with ClockSampler(cx.local) as clk:
        cx.sync()
        e0.record(stream)
        st = run.run(steps)
        e1.record(stream)
        cx.sync()
    ms = cx.max_over_ranks([e0.elapsed_time(e1)])[0]
    _native.check(L.gf_solver_stats(run.handle, C.byref(l1), None, None))
    assert st.status == 0 and st.k + 1 == warmup + steps, (st.status, st.k)
    _native.check(L.gf_solver_profile(run.handle, 1))
    run.run(steps)
    kms = (C.c_double * 8)()
    kcnt = (C.c_int64 * 8)()
    _native.check(L.gf_solver_stats(run.handle, None, kms, kcnt))
    kernels = {KERNEL_NAMES[i]: {"avg_ms": kms[i] / kcnt[i], "count": int(kcnt[i])} for i in range(8) if kcnt[i]}
    es = 4 if setup.dtype == _native.GF_F32 else 8
    # dominant kernel: the pass over this rank's rows of A_hat (fused single
    # pass, or the row pass of the two-pass schedule); algorithmic bytes =
    # m_loc*n*s per launch (the fused pass reads A_hat once; the two-pass
    # schedule's column pass reads it a second time)
    dom = "fused_rowcol_yside" if "fused_rowcol_yside" in kernels else "row_pass_yside"
    alg_bytes = m_loc * n * es
    t_dom = cx.max_over_ranks([kernels[dom]["avg_ms"]])[0] / 1e3
    achieved = alg_bytes / t_dom / 1e9
    peak = peaks["hbm_gbs"]
    out = {"value": steps / (ms / 1e3), "ms_per_step": ms / steps, "steps": steps, "warmup": warmup,
           "kernels": kernels, "gpu_launches": int(l1.value - l0.value), "clocks": clk.summary(),
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": ncu_traffic(dom + ("" if es == 4 else "_f64"), m_loc, n), "kernel": dom,
                        "algorithmic_bytes_per_launch": alg_bytes}}
    if dom == "row_pass_yside" and "col_pass" in kernels:
        # two-pass schedule: the step reads A_hat twice; both passes' bytes
        t2 = t_dom + cx.max_over_ranks([kernels["col_pass"]["avg_ms"]])[0] / 1e3
        out["roofline"]["two_pass_achieved"] = 2 * alg_bytes / t2 / 1e9
    del run, setup
    return out


def e2e_timing(cx, prob, settings, runs=5):
    """The same metric through the public API from HOST buffers: a full
    ``solve(problem)`` on a pinned host copy of this rank's rows of A -- H2D
    of A and the term arrays, equilibration, Gram + Cholesky, iterations to
    eps_rel = 1e-3 and the D2H of x, y, mu, nu -- iterations / wall time,
    max over ranks.  The first call (lazy kernel loading, pool growth) is
    reported as first_solve_s; the value is the best of the rest."""
    import paper_1503_08366_b200 as gf
    from paper_1503_08366_b200 import solver as slv
    torch = cx.torch
    m_loc, n = prob.m, prob.n
    A_pin = torch.empty(tuple(prob.A.shape), dtype=prob.A.dtype, pin_memory=True)
    A_pin.copy_(prob.A)
    prob_pin = gf.GraphFormProblem(A_pin, prob.f, prob.g)
    e2e_runs = []
    for _ in range(runs):
        cx.sync()
        t0 = time.perf_counter()
        res = gf.solve(prob_pin, settings, comm=cx.comm)
        torch.cuda.synchronize()
        e2e_runs.append((cx.max_over_ranks([time.perf_counter() - t0])[0], res))
    e2e_time, res = min(e2e_runs[1:], key=lambda r: r[0]) if len(e2e_runs) > 1 else e2e_runs[-1]
    # phase breakdown of the same public-API path (diagnostic, not the headline)
    cx.sync()
    t0 = time.perf_counter()
    setup_b = gf.prepare(prob_pin, settings, comm=cx.comm)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    run_b = slv._Run(setup_b, prob.f, prob.g, settings, None, None, m_loc)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    run_b.run(0)
    t3 = time.perf_counter()
    run_b.result()
    t4 = time.perf_counter()
    phases = {"prepare_s": t1 - t0, "solver_create_s": t2 - t1, "iterate_s": t3 - t2, "result_s": t4 - t3,
              "iterations": int(run_b.state.iterations)}
    del run_b, setup_b
    h2d = A_pin.numel() * A_pin.element_size() + sum(getattr(prob.f, k).nbytes for k in "abcde") + m_loc \
        + sum(getattr(prob.g, k).nbytes for k in "abcde") + n
    d2h = 8 * (2 * m_loc + 2 * n)
    del A_pin, prob_pin
    return {"value": res.iterations / e2e_time, "unit": "iters/s",
            "h2d_bytes_per_step": int(h2d / max(res.iterations, 1)),
            "d2h_bytes_per_step": int(d2h / max(res.iterations, 1)),
            "time_to_eps_s": e2e_time, "first_solve_s": e2e_runs[0][0], "iterations": res.iterations,
            "status": res.status.value, "objective": res.objective, "setup_s": res.setup_time,
            "h2d_bytes_total": int(h2d), "runs_s": [round(r[0], 4) for r in e2e_runs], "phases": phases}


def run_ours(args):
    import paper_1503_08366_b200 as gf
    cx = Ctx(args)
    torch = cx.torch
    m, n = args.m, args.n
    peaks, peaks_kind = measured_peaks()
    prob, gen_s = device_instance(m, n, cx.rank, cx.world)
    m_loc = prob.m
    fp32 = gf.SolverSettings(precision="fp32")
    e2e = None
    if not args.skip_e2e:
        e2e = e2e_timing(cx, prob, fp32)
        e2e["device_generate_s"] = gen_s
        if cx.world == 1:
            # draw the instance on the GPU and solve it --
            # time to eps with no host generation and no H2D of A
            from paper_1503_08366_b200 import instances
            cx.sync()
            t0 = time.perf_counter()
            pdev, _ = instances.tall_lasso(m, n, 0, dtype=np.float32, device=True)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            rdev = gf.solve(pdev, fp32)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            e2e["device_generated"] = {"generate_s": t1 - t0, "solve_s": t2 - t1, "time_to_eps_s": t2 - t0,
                                       "iterations": rdev.iterations, "status": rdev.status.value}
            del pdev, rdev
    it = iteration_timing(cx, prob, fp32, args.steps, args.warmup, peaks)
    it["roofline"].update({"peak_kind": peaks_kind,
                           # context: the kernel only reads A_hat; a bare TMA read ring on
                           # this part reaches ~7.34 TB/s (profiles/r01_readbw_probe.txt)
                           "read_stream_ceiling_gbs": 7344.0,
                           "frac_of_read_ceiling": it["roofline"]["achieved"] / 7344.0})
    line = {
        "metric": METRIC, "value": it["value"], "unit": "iters/s", "n_gpus": cx.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": it["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference Lasso recipe drawn on the GPU, seed 0, A rounded to fp32)",
        "config": {"workload": f"dense Lasso {m}x{n} fp32 (BASELINE configs[4], 1e9 coefficients)",
                   "m": m, "n": n,
                   "parallelism": f"row partition x{cx.world}" + (" (NCCL all-reduce)" if cx.use_comm else ""),
                   "rows_per_rank": m_loc, "l2": "A is 4 GB >> 126 MB L2; no flush needed"},
        "e2e": e2e, "roofline": it["roofline"], "kernels": it["kernels"], "gpu_launches": it["gpu_launches"],
        "clocks": it["clocks"],
    }
    if not args.no_fp64:
        # the reference's own precision: the same instance, fp64 matrix passes
        # (A_hat 8 GB, G^-1 200 MB) -- the like-for-like line for the
        # reference arm's fp64 CPU numbers
        st64 = gf.SolverSettings(precision="fp64")
        k64 = max(1, min(args.steps, 300))
        it64 = iteration_timing(cx, prob, st64, k64, args.warmup, peaks)
        fp64 = {"value": it64["value"], "unit": "iters/s", "ms_per_step": it64["ms_per_step"], "steps": k64,
                "warmup": args.warmup, "dtype": "f64", "roofline": it64["roofline"], "kernels": it64["kernels"],
                "gpu_launches": it64["gpu_launches"], "clocks": it64["clocks"]}
        if not args.skip_e2e:
            fp64["e2e"] = e2e_timing(cx, prob, st64, runs=3)
        line["fp64"] = fp64
    if not args.no_cpu and cx.world == 1:
        # the oracle port on the FULL instance (the same code as the reference
        # arm), 5 timed iterations after 2 warm-up: ~15 s of host work
        A_host = prob.A.cpu().numpy()
        val, t_setup = time_port(A_host, prob.f, prob.g, 5, 2)
        del A_host
        line["cpu_baseline"] = {"value": val, "unit": "iters/s", "cores": host_cores(), "kind": "port",
                                "sample": f"full {m}x{n} instance (fp32-rounded A in fp64, as the reference "
                                          f"arm); prepare {t_setup:.1f}s excluded; 5 iterations after 2 warm-up"}
    if cx.rank == 0:
        print(json.dumps(line), flush=True)
    del prob
    cx.close()
    return 0


def relaunch_under_torchrun(args):
    """--gpus N without a torchrun environment: re-exec this command as N
    ranks (one process per GPU) on 127.0.0.1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=M_FULL)
    ap.add_argument("--n", type=int, default=N_FULL)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 (reference precision) sub-line")
    ap.add_argument("--skip-e2e", action="store_true",
                    help="profiling runs only: skip the end-to-end solves (the line then has e2e null)")
    ap.add_argument("--force-comm", action="store_true",
                    help="use the NCCL row-partition path even on one GPU (checks the multi-GPU plumbing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

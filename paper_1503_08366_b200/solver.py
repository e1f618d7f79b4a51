"""ADMM graph-form solver, drop-in for the reference ``solver.py``.

``prepare`` / ``solve`` keep the reference signatures, defaults, validation
and result semantics (solver.py:52-437).  The loop itself runs on the GPU:
``gf_solver_run`` launches chunks of iterations whose stop rule, degenerate
checks and adaptive-rho decisions are taken by a device-side controller
(csrc/gf_solver.cu), so a solve needs no per-iteration host round trip.  When
a ``callback``, ``trace`` or ``verbose`` is requested the host steps one
iteration at a time and reads the recorded iteration back, so the observable
per-iteration values are the same.

Extension (not in the reference): ``SolverSettings.precision`` selects the
arithmetic type of the matrix passes -- "fp64" (also what None means: the
reference computes in float64 whatever the input, problem.py:35) or "fp32"
(opt-in: A_hat and G^-1 stored and streamed in fp32).  Term math, norms and
the stopping rule are fp64 in both.
"""

from __future__ import annotations

import ctypes as C
import enum
import time
import weakref
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native
from .equilibration import Equilibration
from .errors import DimensionError, ParameterError
from .problem import GraphFormProblem, duality_gap
from .projection import ProjectorCache, _dtype_for

__all__ = ["Status", "SolverSettings", "SolveResult", "Setup", "IterationSnapshot", "prepare",
           "solve", "recover_duals", "unscale", "residual_stop", "gap_stop", "adapt_rho"]


class Status(enum.Enum):
    SOLVED = "Solved"
    MAX_ITERATIONS = "MaxIterations"
    DEGENERATE = "Degenerate"


_STATUS = {1: Status.SOLVED, 2: Status.MAX_ITERATIONS, 3: Status.DEGENERATE}


@dataclass(frozen=True)
class SolverSettings:
    """Outer-loop knobs (solver.py:52-92) plus ``precision``."""

    rho0: float = 1.0
    abs_tol: float = 1e-4
    rel_tol: float = 1e-3
    max_iter: int = 10_000
    alpha: float = 1.7
    adaptive_rho: bool = True
    delta: float = 1.05
    tau: float = 0.8
    equilibrate: bool = True
    gap_stop: bool = False
    projection: str = "direct"
    projection_tol: Optional[float] = None
    max_inner: Optional[int] = None
    verbose: bool = False
    precision: Optional[str] = None

    def __post_init__(self):
        if not self.rho0 > 0.0:
            raise ParameterError("rho0 must be positive")
        if not self.abs_tol > 0.0 or not self.rel_tol > 0.0:
            raise ParameterError("tolerances must be positive")
        if self.max_iter < 1:
            raise ParameterError("max_iter must be at least 1")
        if not 0.0 < self.alpha < 2.0:
            raise ParameterError("alpha must lie in (0, 2)")
        if not self.delta > 1.0:
            raise ParameterError("delta must exceed 1")
        if not 0.0 < self.tau <= 1.0:
            raise ParameterError("tau must lie in (0, 1]")
        if self.projection not in ("direct", "indirect"):
            raise ParameterError("projection must be 'direct' or 'indirect'")
        if self.projection_tol is not None and not self.projection_tol > 0.0:
            raise ParameterError("projection_tol must be positive")
        if self.precision not in (None, "fp32", "fp64", "float32", "float64"):
            raise ParameterError("precision must be None, 'fp32' or 'fp64'")


@dataclass
class SolveResult:
    x: np.ndarray
    y: np.ndarray
    mu: np.ndarray
    nu: np.ndarray
    objective: float
    primal_residual: float
    dual_residual: float
    gap: Optional[float]
    status: Status
    iterations: int
    solve_time: float
    setup_time: float
    final_rho: float


@dataclass
class IterationSnapshot:
    """Hat-space view of one iteration (solver.py:123-139)."""

    k: int
    rho: float
    x_hat: np.ndarray
    y_hat: np.ndarray
    xt: np.ndarray
    yt: np.ndarray
    x_half_hat: np.ndarray
    y_half_hat: np.ndarray
    r_pri: float
    r_dual: float
    eps_pri: float
    eps_dual: float
    inner_iterations: int = 0


class Setup:
    """Device-resident pre-conditioning + projector, reusable across solves
    on the same matrix (solver.py:112-120).  ``A_hat`` is downloaded on
    first access; the solve never needs it on the host."""

    def __init__(self, handle, m, n, mode, tol, max_inner, dtype, comm=None):
        self.handle = handle
        self.m, self.n = m, n
        self.dtype = dtype
        self.comm = comm
        info = _native.SetupInfo()
        L = _native.lib()
        _native.check(L.gf_setup_get_info(handle, C.byref(info)))
        d = np.empty(m)
        e = np.empty(n)
        _native.check(L.gf_setup_scaling(handle, _native.ptr(d), _native.ptr(e), _native.stream()))
        self.scaling = Equilibration(d=d, e=e, p=2, gamma=info.gamma, iterations=int(info.sweeps),
                                     converged=bool(info.converged))
        self.setup_time = float(info.setup_seconds)
        ph = C.c_void_p()
        _native.check(L.gf_setup_projector(handle, C.byref(ph)))
        mh = C.c_void_p()
        _native.check(L.gf_setup_matrix(handle, C.byref(mh)))
        self._mview = _MatrixView(mh, m, n)
        # the projector view holds this Setup (its owner); the Setup keeps only a
        # weak reference back, so dropping the Setup frees the device memory at
        # once instead of at the next cyclic garbage collection
        self._proj_args = (ph, mode, m, n, tol, max_inner)
        self._proj_ref = None
        self._A_hat = None

    @property
    def projector(self) -> ProjectorCache:
        p = self._proj_ref() if self._proj_ref is not None else None
        if p is None:
            ph, mode, m, n, tol, max_inner = self._proj_args
            p = ProjectorCache(ph, self._mview, mode, m, n, tol, max_inner, owner=self)
            self._proj_ref = weakref.ref(p)
        return p

    @property
    def A_hat(self):
        if self._A_hat is None:
            self._A_hat = self._mview.download()
        return self._A_hat

    def __del__(self):
        try:
            if self.handle:
                _native.load_library().gf_setup_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class _MatrixView:
    def __init__(self, handle, m, n):
        self.handle, self.m, self.n = handle, m, n

    def download(self):
        out = np.empty((self.m, self.n))
        _native.check(_native.lib().gf_matrix_download(self.handle, _native.ptr(out), _native.stream()))
        return out


def _global_rows(m_local: int) -> int:
    """Sum of the ranks' row counts over the default torch.distributed group
    (the group the communicator was built from)."""
    import torch
    import torch.distributed as dist
    dev = _native.device() if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([m_local], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    return int(t.item())


def prepare(problem: GraphFormProblem, settings: SolverSettings = None,
            scaling: Optional[Equilibration] = None, comm=None) -> Setup:
    """Equilibrate (unless disabled or supplied), scale A in place on the
    device and build the projector (solver.py:148-169)."""
    if settings is None:
        settings = SolverSettings()
    L = _native.lib()
    t0 = time.perf_counter()
    A = problem.A
    m, n = problem.m, problem.n
    dt = _dtype_for(A, settings.precision)
    M = _native.Matrix(A, dt)
    tol = settings.projection_tol if settings.projection_tol is not None else 1e-8
    if settings.max_inner is not None:
        max_inner = settings.max_inner
    else:   # projection.py:146 on the GLOBAL row count (every rank the same CGLS cap)
        mg = m if comm is None else _global_rows(m)
        max_inner = max(100, 2 * min(mg, n))
    d_in = e_in = None
    if scaling is not None:
        if scaling.d.shape != (m,) or scaling.e.shape != (n,):
            raise DimensionError("scaling does not match the matrix shape")
        d_in = np.ascontiguousarray(scaling.d, dtype=float)
        e_in = np.ascontiguousarray(scaling.e, dtype=float)
    h = C.c_void_p()
    _native.check(L.gf_setup_create(
        M.handle, 1 if settings.equilibrate else 0,
        None if d_in is None else _native.ptr(d_in), None if e_in is None else _native.ptr(e_in),
        0 if settings.projection == "direct" else 1, float(tol), int(max_inner),
        None if comm is None else comm.handle, _native.stream(), C.byref(h)))
    M.release()  # the setup owns the matrix now
    S = Setup(h, m, n, settings.projection, tol, max_inner, dt, comm)
    S.setup_time = time.perf_counter() - t0
    return S


def _gf_settings(s: SolverSettings):
    return _native.Settings(
        rho0=float(s.rho0), abs_tol=float(s.abs_tol), rel_tol=float(s.rel_tol),
        max_iter=int(s.max_iter), alpha=float(s.alpha), adaptive_rho=1 if s.adaptive_rho else 0,
        delta=float(s.delta), tau=float(s.tau), projection=0 if s.projection == "direct" else 1,
        projection_tol=float(s.projection_tol) if s.projection_tol is not None else -1.0,
        gap_stop=1 if s.gap_stop else 0)


_VERBOSE_HEADER = (f"{'iter':>6} {'r_pri':>11} {'eps_pri':>11} {'r_dual':>11} "
                   f"{'eps_dual':>11} {'rho':>10} {'objective':>13}")


class _Run:
    """One device solver instance (gf_solver)."""

    def __init__(self, setup: Setup, f, g, settings, x0, nu0, m_local):
        L = _native.lib()
        self.L = L
        self.setup = setup
        self.m, self.n = m_local, setup.n
        fT, self._fk = _native.host_terms(f)
        gT, self._gk = _native.host_terms(g)
        self._x0 = None if x0 is None else np.ascontiguousarray(np.asarray(x0, float))
        self._nu0 = None if nu0 is None else np.ascontiguousarray(np.asarray(nu0, float))
        if self._x0 is not None and self._x0.shape != (self.n,):
            raise DimensionError("x0 must have length n")
        if self._nu0 is not None and self._nu0.shape != (self.m,):
            raise DimensionError("nu0 must have length m")
        self.gs = _gf_settings(settings)
        h = C.c_void_p()
        _native.check(L.gf_solver_create(
            setup.handle, C.byref(fT), C.byref(gT), C.byref(self.gs),
            None if self._x0 is None else _native.ptr(self._x0),
            None if self._nu0 is None else _native.ptr(self._nu0), _native.stream(), C.byref(h)))
        self.handle = h
        self.state = _native.SolverState()

    def run(self, steps=0):
        _native.check(self.L.gf_solver_run(self.handle, int(steps), C.byref(self.state), _native.stream()))
        return self.state

    def history(self, count):
        out = np.empty((max(count, 1), 6))
        _native.check(self.L.gf_solver_history(self.handle, int(count), _native.ptr(out), _native.stream()))
        return out[:count]

    def snapshot(self):
        bufs = [np.empty(k) for k in (self.n, self.m, self.n, self.m, self.n, self.m)]
        _native.check(self.L.gf_solver_snapshot(self.handle, *(_native.ptr(b) for b in bufs), _native.stream()))
        return bufs

    def result(self):
        x, mu = np.empty(self.n), np.empty(self.n)
        y, nu = np.empty(self.m), np.empty(self.m)
        _native.check(self.L.gf_solver_result(self.handle, _native.ptr(x), _native.ptr(y), _native.ptr(mu),
                                              _native.ptr(nu), C.byref(self.state), _native.stream()))
        return x, y, mu, nu, self.state

    def elapsed_ms(self):
        v = C.c_double()
        _native.check(self.L.gf_solver_elapsed_ms(self.handle, C.byref(v)))
        return float(v.value)

    def __del__(self):
        try:
            if self.handle:
                self.L.gf_solver_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def solve(problem: GraphFormProblem, settings: SolverSettings = None, *,
          x0=None, nu0=None, scaling: Optional[Equilibration] = None,
          setup: Optional[Setup] = None, callback: Optional[Callable] = None,
          trace: Optional[list] = None, comm=None) -> SolveResult:
    """Solve minimize f(y) + g(x) s.t. y = A x (solver.py:248-437).

    ``comm`` (extension): a ``distributed.Comm`` when ``problem`` holds this
    rank's rows of a row-partitioned problem (see ``distributed.py``)."""
    if settings is None:
        settings = SolverSettings()
    own = setup is None
    if own:
        setup = prepare(problem, settings, scaling=scaling, comm=comm)
    setup_time = setup.setup_time if own else 0.0
    t0 = time.perf_counter()
    run = _Run(setup, problem.f, problem.g, settings, x0, nu0, problem.m)
    observe = callback is not None or trace is not None or settings.verbose
    if settings.verbose:
        print(_VERBOSE_HEADER)
    if not observe:
        run.run(0)
    else:
        seen = -1
        first = len(trace) if trace is not None else 0   # snapshots of THIS solve start here
        indirect = settings.projection == "indirect"
        wide = problem.m < problem.n
        while True:
            st = run.run(1)
            # a step begins with the (indirect) projection of the previous
            # iteration: its CGLS count belongs to the previous snapshot
            # (solver.py:410-411) -- also when that step records nothing new
            # (the projection of the last iteration, or a degenerate one)
            if trace is not None and len(trace) > first and indirect and not wide:
                trace[-1].inner_iterations = int(st.inner_iterations)
            if st.k > seen:
                k = int(st.k)
                seen = k
                r_pri, r_dual, eps_pri, eps_dual, rho, obj = run.history(k + 1)[k]
                if callback is not None:
                    callback(k, r_pri, r_dual, eps_pri, eps_dual, rho, obj)
                if settings.verbose:
                    print(f"{k:6d} {r_pri:11.4e} {eps_pri:11.4e} {r_dual:11.4e} "
                          f"{eps_dual:11.4e} {rho:10.3e} {obj:13.6e}")
                if trace is not None:
                    xk, yk, xt, yt, xhh, yhh = run.snapshot()
                    trace.append(IterationSnapshot(k=k, rho=float(rho), x_hat=xk, y_hat=yk, xt=xt, yt=yt,
                                                   x_half_hat=xhh, y_half_hat=yhh, r_pri=float(r_pri),
                                                   r_dual=float(r_dual), eps_pri=float(eps_pri),
                                                   eps_dual=float(eps_dual), inner_iterations=0))
                    # wide: the step that records iteration k also ran its
                    # projection, unless iteration k stopped the solve
                    if indirect and wide and st.status != 1:
                        trace[-1].inner_iterations = int(st.inner_iterations)
            if st.status != 0:
                break
    x, y, mu, nu, st = run.result()
    return SolveResult(
        x=x, y=y, mu=mu, nu=nu, objective=float(st.objective),
        primal_residual=float(st.r_pri), dual_residual=float(st.r_dual),
        gap=float(st.gap) if st.gap_valid else None,
        status=_STATUS[st.status], iterations=int(st.iterations),
        solve_time=time.perf_counter() - t0, setup_time=setup_time, final_rho=float(st.final_rho))


# ----------------------------------------------------- standalone helpers --
# The solve fuses these into its kernels; the standalone versions keep the
# reference's public helpers (solver.py:172-239) and run on the device.
def _dev(*xs):
    return [_native.to_device64(x) for x in xs]


def recover_duals(x_prev, y_prev, xt, yt, x_half, y_half, rho):
    """(mu_half, nu_half, mu, nu) of one iteration (solver.py:172-183)."""
    a = _dev(x_prev, y_prev, xt, yt, x_half, y_half)
    xp, yp, xtt, ytt, xh, yh = a
    out = (-rho * (xh - xp + xtt), -rho * (yh - yp + ytt), -rho * xtt, -rho * ytt)
    return tuple(_native.like_input(o, r) for o, r in zip(out, (x_half, y_half, xt, yt)))


def unscale(x_hat, y_hat, mu_hat, nu_hat, d, e):
    """Hat space -> original variables (solver.py:186-188)."""
    xh, yh, mh, nh, dd, ee = _dev(x_hat, y_hat, mu_hat, nu_hat, d, e)
    out = (ee * xh, yh / dd, mh / ee, dd * nh)
    return tuple(_native.like_input(o, r) for o, r in zip(out, (x_hat, y_hat, mu_hat, nu_hat)))


def residual_stop(A, x_half, y_half, mu_half, nu_half, eps_abs, eps_rel):
    """(stop, eps_pri, eps_dual, r_pri, r_dual) in the original space
    (solver.py:191-202); the two matvecs run through gf_matvec."""
    import torch
    M = _native.Matrix(A, _dtype_for(A, None))
    L = _native.lib()
    xh, yh, mh, nh = _dev(x_half, y_half, mu_half, nu_half)
    ax = torch.empty(M.m, dtype=torch.float64, device=xh.device)
    atn = torch.empty(M.n, dtype=torch.float64, device=xh.device)
    _native.check(L.gf_matvec(M.handle, 0, _native.ptr(xh), _native.ptr(ax), _native.stream()))
    _native.check(L.gf_matvec(M.handle, 1, _native.ptr(nh), _native.ptr(atn), _native.stream()))
    r_pri = float(torch.linalg.vector_norm(ax - yh))
    r_dual = float(torch.linalg.vector_norm(atn + mh))
    eps_pri = eps_abs + eps_rel * float(torch.linalg.vector_norm(yh))
    eps_dual = eps_abs + eps_rel * float(torch.linalg.vector_norm(mh))
    return (r_pri <= eps_pri and r_dual <= eps_dual, eps_pri, eps_dual, r_pri, r_dual)


def gap_stop(problem, x_full, y_full, mu_full, nu_full, eps_abs, eps_rel):
    """Gap-based stopping test at the full iterate (solver.py:205-218):
    ``(stop, gap)``; ``gap`` is None when a conjugate is unsupported and an
    infinite gap never stops.  The solve runs this test inside its device
    controller; this is the standalone form (conjugates on the GPU)."""
    gap = duality_gap(problem, x_full, y_full, mu_full, nu_full)
    if gap is None or not np.isfinite(gap):
        return False, gap
    obj = problem.objective(x_full, y_full)
    if not np.isfinite(obj):
        return False, gap
    return gap <= eps_abs + eps_rel * abs(obj), gap


def adapt_rho(rho, xt, yt, k, l, u, r_pri, r_dual, eps_pri, eps_dual, delta, tau):
    """One adaptive-penalty decision (solver.py:221-239, Alg. 3)."""
    if r_dual < eps_dual and tau * k > l:
        new_rho = delta * rho
        ratio = rho / new_rho
        a, b = _dev(xt, yt)
        return new_rho, _native.like_input(a * ratio, xt), _native.like_input(b * ratio, yt), l, k
    if r_pri < eps_pri and tau * k > u:
        new_rho = rho / delta
        ratio = rho / new_rho
        a, b = _dev(xt, yt)
        return new_rho, _native.like_input(a * ratio, xt), _native.like_input(b * ratio, yt), k, u
    return rho, xt, yt, l, u

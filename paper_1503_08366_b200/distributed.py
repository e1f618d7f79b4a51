"""Row-partitioned multi-GPU solves: one process per GPU.

A tall problem (m >= n) is split into contiguous row blocks, one per rank:
rank r holds A[r0:r1], f[r0:r1] and the matching y-side vectors; g, the x
side, the factor of I + A'A and the rho state are replicated.  The CUDA
library owns an NCCL communicator (built from a unique id that rank 0 creates
and ``torch.distributed`` broadcasts) and issues

  setup      one all-reduce per Sinkhorn sweep (n column sums + scalars),
             one for the Frobenius rescale, one of the Gram matrix (packed
             lower triangle);
  iteration  ONE all-reduce of 2*ld + 8 doubles between the column pass and
             the controller: [A_hat' c_y | A_hat' nu^ | r_pri^2, ||y||^2,
             f(y), drift, flags, and the two gap terms]; every rank then
             takes the same decision.

Usage (under torchrun, after ``torch.distributed.init_process_group``)::

    comm = distributed.init_comm()
    r0, r1 = distributed.row_range(m, comm.rank, comm.world)
    res = distributed.solve_sharded(A[r0:r1], f.slice(r0, r1), g, comm=comm)

``res.x`` / ``res.mu`` are the full (replicated) vectors, ``res.y`` /
``res.nu`` this rank's rows; objective and residuals are global.
"""

from __future__ import annotations

import ctypes as C

from . import _native
from .errors import DimensionError
from .functions import SeparableFunction
from .problem import GraphFormProblem

__all__ = ["Comm", "init_comm", "row_range", "solve_sharded", "prepare_sharded"]


class Comm:
    """Owning handle of the library's NCCL communicator."""

    def __init__(self, handle, rank: int, world: int):
        self.handle = handle
        self.rank = rank
        self.world = world

    def __del__(self):
        try:
            if self.handle:
                _native.load_library().gf_comm_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def row_range(m: int, rank: int, world: int):
    """Contiguous, balanced row block [r0, r1) of ``rank`` (same rule as the
    fused kernel's per-CTA split)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return m * rank // world, m * (rank + 1) // world


def _broadcast_id(uid: bytes, group=None) -> bytes:
    import torch.distributed as dist
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_comm(group=None) -> Comm:
    """NCCL communicator over the ranks of the default torch.distributed group
    (any backend: the id travels with broadcast_object_list)."""
    import torch.distributed as dist
    L = _native.lib()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = b""
    if rank == 0:
        buf = C.create_string_buffer(128)
        _native.check(L.gf_comm_unique_id(buf))
        uid = buf.raw
    uid = _broadcast_id(uid, group)
    h = C.c_void_p()
    _native.check(L.gf_comm_create(C.c_char_p(uid), world, rank, C.byref(h)))
    return Comm(h, rank, world)


def prepare_sharded(A_local, f_local: SeparableFunction, g: SeparableFunction, settings=None,
                    comm: Comm = None, scaling=None):
    from .solver import prepare
    problem = GraphFormProblem(A_local, f_local, g)
    return prepare(problem, settings, scaling=scaling, comm=comm)


def solve_sharded(A_local, f_local: SeparableFunction, g: SeparableFunction, settings=None, *,
                  comm: Comm = None, x0=None, nu0=None, setup=None, callback=None):
    """solve() over this rank's rows; every rank must call it collectively."""
    from .solver import solve
    if len(f_local) != A_local.shape[0]:
        raise DimensionError("f_local must have one term per local row")
    problem = GraphFormProblem(A_local, f_local, g)
    return solve(problem, settings, x0=x0, nu0=nu0, setup=setup, callback=callback, comm=comm)

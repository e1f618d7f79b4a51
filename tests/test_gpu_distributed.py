"""GPU: the row-partitioned path through a real NCCL communicator.

The round's boxes have one GPU, and NCCL refuses two ranks on one device, so
the communicator here has ONE rank: every collective call site of the
library (Sinkhorn sweeps, rescale, Gram, per-iteration payload, CGLS dots)
runs through NCCL, and the results must equal the communicator-free solve
bit for bit (a one-rank all-reduce is a copy).  The multi-rank decomposition
itself is checked on CPU (test_distributed_cpu.py, world size 2).
"""

import numpy as np
import pytest
import torch.distributed as dist

import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import distributed
from tests import _cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(tmp_path_factory):
    store = dist.FileStore(str(tmp_path_factory.mktemp("pg") / "store"), 1)
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    c = distributed.init_comm()
    yield c
    del c
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["lasso_tall_1000x200", "svm_2000x100", "lasso_tall_1000x200_indirect",
                                  "huber_fit_400x80", "lp_600x240_r32"])
def test_one_rank_comm_equals_plain_solve(comm, name):
    fx = _cases.load("solve_" + name)
    prob = _cases.build_problem(fx, as_float32=name.endswith("_r32"))
    st = gf.SolverSettings(precision="fp32" if name.endswith("_r32") else None, **_cases.settings_of(fx))
    a = gf.solve(prob, st)
    r0, r1 = distributed.row_range(prob.m, comm.rank, comm.world)
    b = distributed.solve_sharded(prob.A[r0:r1], prob.f.slice(r0, r1), prob.g, st, comm=comm)
    assert b.status == a.status and b.iterations == a.iterations
    for k in ("x", "y", "mu", "nu"):
        np.testing.assert_array_equal(getattr(b, k), getattr(a, k), err_msg=k)
    assert b.objective == a.objective
    if not name.endswith("_r32"):
        assert b.iterations == int(fx["iterations"])


def test_comm_rejects_wide(comm):
    fx = _cases.load("solve_lasso_wide_200x1000")
    prob = _cases.build_problem(fx)
    with pytest.raises(NotImplementedError, match="tall"):
        distributed.solve_sharded(prob.A, prob.f, prob.g, comm=comm)

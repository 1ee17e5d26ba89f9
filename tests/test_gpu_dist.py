"""GPU: the time-partitioned hierarchy over a real NCCL process group of
one rank (the pool gives one GPU per call; world sizes 2 and 4 are covered
over gloo on CPU in test_dist_gloo.py).  Exercises the CUDA-tensor paths of
the collectives (all_gather, gather, scatter, batched P2P) and checks the
result against the single-GPU hierarchy bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2104_09404_b200 as P
from paper_2104_09404_b200.distributed import DistMgritHierarchy, mgrit_solve_distributed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("L,m,cycle", [(2, 4, "v"), (4, 2, "f")])
def test_nccl_world1_equals_single(nccl_group, L, m, cycle):
    pb = P.Problem(name="d", n_x=64, n_t=64, cfl=0.1, n_modes=3, n_levels=L, m=m, cycle=cycle,
                   max_iters=3)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    ref = P.serial.march(st[0], u0, pb.n_t)
    traj, rec = P.mgrit_solve(st, u0, tg, pb.space_grid(), pb.options(), reference=ref)
    dtraj, drec = mgrit_solve_distributed(st, u0, tg, pb.space_grid(), pb.options(),
                                          reference=ref)
    assert np.array_equal(dtraj.values, traj.values)
    np.testing.assert_allclose(drec.residuals, rec.residuals, rtol=1e-12)
    np.testing.assert_allclose(drec.errors, rec.errors, rtol=1e-12)
    h = DistMgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    g = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    for obj in (h, g):
        obj.relax(0)
        obj.restrict(0)
    assert torch.equal(h.level_values(1), g.levels[1].u)

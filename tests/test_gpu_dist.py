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


def test_nccl_world1_relax_fine_values_is_the_fused_kernel(nccl_group):
    """The distributed bench step runs the N = 1 fused FCF kernel: same
    trajectory bit for bit, and one fcf launch + no extra sweeps at world 1."""
    pb = P.Problem(name="d", n_x=128, n_t=256, cfl=0.2, n_modes=3, n_levels=2, m=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    c = P.serial.march(st[0], u0, pb.n_t)[::4, 0]
    h = DistMgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    g = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    h.load_c_points(c)
    g.load_c_points(c)
    assert h._fcf_workspace() is not None
    n0 = P._lib.launch_count()
    got = h.relax_fine_values()
    assert P._lib.launch_count() - n0 == 1
    want = g.relax_fine_values()
    assert torch.equal(got, want.reshape(got.shape))
    assert torch.equal(h.c_points() if hasattr(h, "c_points") else h._c[h._cur],
                       g._c[g._cur])


def test_nccl_world1_relax_to_host(nccl_group):
    """The N > 1 bench's end-to-end step: one launch on mapped pinned buffers,
    same rows as relax_fine_values."""
    pb = P.Problem(name="d", n_x=128, n_t=256, cfl=0.2, n_modes=3, n_levels=2, m=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    c = P.serial.march(st[0], u0, pb.n_t)[::4, 0]
    h = DistMgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    g = DistMgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    c_host = c.cpu().pin_memory()
    out = torch.empty(pb.n_t + 1, pb.n_x, dtype=torch.float64).pin_memory()
    h.relax_to_host(c_host, out)
    torch.cuda.synchronize()
    g.load_c_points(c)
    want = g.relax_fine_values()
    assert torch.equal(out, want.reshape(out.shape).cpu())
    assert torch.equal(h._c[h._cur], g._c[g._cur])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker2(rank, world, port, outdir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2104_09404_b200 as P2
        from paper_2104_09404_b200.distributed import (DistMgritHierarchy as DH,
                                                       mgrit_solve_distributed as msd)
        pb = P2.Problem(name="d2", n_x=128, n_t=512, cfl=0.1, n_modes=3, n_levels=3, m=4,
                        max_iters=3)
        u0 = pb.initial_state()
        tg = pb.time_grid(u0)
        st = pb.steppers(tg)
        ref = P2.serial.march(st[0], u0, pb.n_t)
        traj, rec = msd(st, u0, tg, pb.space_grid(), pb.options(), reference=ref)
        h = DH(st, u0, tg, pb.space_grid(), pb.options())
        h.load_c_points(ref[::4, 0][h.off[0]: h.off[0] + h.nloc[0] + 1])
        local = h.relax_fine_values().cpu()
        torch.save({"rank": rank, "off": h.off[0], "n0": h.nloc[0], "local": local,
                    "traj": None if traj is None else torch.from_numpy(traj.values),
                    "res": rec.residuals.tolist(), "err": rec.errors.tolist(),
                    "div": rec.diverged_at}, os.path.join(outdir, f"r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NCCL over NVLink)")
def test_nccl_world2_equals_single(tmp_path):
    """Two ranks over NCCL: the solve and the fused distributed relaxation
    equal the single-GPU ones bit for bit (iterates) / to 1e-12 (norms)."""
    import torch.multiprocessing as mp
    mp.spawn(_worker2, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    pb = P.Problem(name="d2", n_x=128, n_t=512, cfl=0.1, n_modes=3, n_levels=3, m=4,
                   max_iters=3)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    ref = P.serial.march(st[0], u0, pb.n_t)
    traj, rec = P.mgrit_solve(st, u0, tg, pb.space_grid(), pb.options(), reference=ref)
    g = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    g.load_c_points(ref[::4, 0])
    whole = g.relax_fine_values().cpu().reshape(pb.n_t + 1, -1)
    r0 = torch.load(tmp_path / "r0.pt")
    assert np.array_equal(r0["traj"].numpy(), traj.values)
    np.testing.assert_allclose(r0["res"], rec.residuals, rtol=1e-12)
    np.testing.assert_allclose(r0["err"], rec.errors, rtol=1e-12)
    for r in range(2):
        d = torch.load(tmp_path / f"r{r}.pt")
        lo = d["off"] * 4
        assert torch.equal(d["local"], whole[lo: lo + d["n0"] * 4 + 1]), r

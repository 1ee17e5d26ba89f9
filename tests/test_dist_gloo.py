"""CPU, world_size 2 and 4 over gloo: the time-partitioned hierarchy
(paper_2104_09404_b200/distributed.py) reproduces the single-process
hierarchy bit for bit (iterates) and to 1e-12 (norms), with the mgp_sweep
emulator standing in for the kernels (tests/sweep_emulator.py)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(n_t, m, L, cycle="v", relax="fcf", guess="last-step", iters=3):
    import paper_2104_09404_b200 as P
    return P.Problem(name="dist", n_x=16, n_t=n_t, cfl=0.1, n_modes=2, weno_order=(5,),
                     stepper=("ssprk3",), n_levels=L, m=m, cycle=cycle, relaxation=relax,
                     guess=guess, max_iters=iters)


def _worker(rank, world, port, case, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OPENBLAS_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sweep_emulator
        sweep_emulator.install()
        import paper_2104_09404_b200 as P
        from paper_2104_09404_b200.distributed import (DistMgritHierarchy,
                                                       mgrit_solve_distributed)
        pb = _problem(**case)
        u0 = pb.initial_state()
        tg = pb.time_grid(u0)
        steppers = pb.steppers(tg)
        ref = P.serial.march(steppers[0], u0, pb.n_t)
        # 1) whole solve
        traj, rec = mgrit_solve_distributed(steppers, u0, tg, pb.space_grid(), pb.options(),
                                            reference=ref)
        # 2) level operations one by one
        h = DistMgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
        seq = ["f0", "c0", "f0", "r0", "c1", "r1", "i1", "i0", "c0", "c0", "r0", "i0"]
        snaps = []
        for op in seq:
            l = int(op[1])
            getattr(h, {"f": "f_relax", "c": "c_relax", "r": "restrict",
                        "i": "interpolate"}[op[0]])(l)
            if op[0] == "r" and l + 1 == pb.n_levels - 1:
                h.coarse_solve()
            v0 = h.fine_values()
            v1 = h.level_values(1)
            res = h.residual_norm()
            if rank == 0:
                snaps.append((op, v0.numpy().copy(), v1.numpy().copy(), res))
        if rank == 0:
            np.save(os.path.join(outdir, "traj.npy"), traj.values)
            np.save(os.path.join(outdir, "resid.npy"), rec.residuals)
            np.save(os.path.join(outdir, "err.npy"), rec.errors)
            np.save(os.path.join(outdir, "div.npy"), np.array([-1 if rec.diverged_at is None
                                                               else rec.diverged_at]))
            torch.save(snaps, os.path.join(outdir, "snaps.pt"))
    finally:
        dist.destroy_process_group()


def _single(case):
    import sweep_emulator
    import paper_2104_09404_b200 as P
    sweep_emulator.install()
    try:
        pb = _problem(**case)
        u0 = pb.initial_state()
        tg = pb.time_grid(u0)
        steppers = pb.steppers(tg)
        ref = P.serial.march(steppers[0], u0, pb.n_t)
        traj, rec = P.mgrit_solve(steppers, u0, tg, pb.space_grid(), pb.options(),
                                  reference=ref)
        h = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
        seq = ["f0", "c0", "f0", "r0", "c1", "r1", "i1", "i0", "c0", "c0", "r0", "i0"]
        snaps = []
        for op in seq:
            l = int(op[1])
            getattr(h, {"f": "f_relax", "c": "c_relax", "r": "restrict",
                        "i": "interpolate"}[op[0]])(l)
            if op[0] == "r" and l + 1 == pb.n_levels - 1:
                h.coarse_solve()
            snaps.append((op, h.fine_values().numpy().copy(), h.levels[1].u.numpy().copy(),
                          h.residual_norm()))
        return traj, rec, snaps
    finally:
        sweep_emulator.remove()


CASES = [
    (2, dict(n_t=64, m=2, L=4)),                         # every level distributed
    (2, dict(n_t=32, m=4, L=3, relax="f", guess="injection")),
    (4, dict(n_t=32, m=2, L=4, cycle="f")),              # level 2 agglomerated on rank 0
    (2, dict(n_t=16, m=2, L=3)),
]


@pytest.mark.parametrize("world,case", CASES)
def test_distributed_equals_single(tmp_path, world, case):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True)
    traj, rec, snaps = _single(case)
    assert np.array_equal(np.load(tmp_path / "traj.npy"), traj.values)
    np.testing.assert_allclose(np.load(tmp_path / "resid.npy"), rec.residuals, rtol=1e-12)
    np.testing.assert_allclose(np.load(tmp_path / "err.npy"), rec.errors, rtol=1e-12)
    dsnaps = torch.load(tmp_path / "snaps.pt", weights_only=False)
    for (op, a0, a1, ra), (_, b0, b1, rb) in zip(dsnaps, snaps):
        assert np.array_equal(a0, b0), op
        assert np.array_equal(a1, b1), op
        np.testing.assert_allclose(ra, rb, rtol=1e-12)


def test_partition_rules():
    from paper_2104_09404_b200.distributed import partition
    assert partition(65536, 4, 7, 8) == (6, [2048, 512, 128, 32, 8, 2])
    assert partition(262144, 16, 5, 8) == (3, [2048, 128, 8])
    assert partition(4096, 4, 2, 8) == (1, [128])
    from paper_2104_09404_b200 import ConfigError
    with pytest.raises(ConfigError):
        partition(12, 2, 2, 4)

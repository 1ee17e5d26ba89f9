"""GPU parity of the MGRIT hierarchy (C-points-only finest storage, fused
level kernels) against the reference's own histories (golden fixtures) and
the oracle restatement of mgrit.py.

Tolerances (north_star): residual and error histories within 1e-10
relative, identical divergence iteration, trajectories bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import paper_2104_09404_b200 as P
from oracle import mgrit_oracle

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def _problem(spec, data):
    u0 = data[spec["name"] + "__u0"]
    sg = P.SpatialGrid(spec.get("length", 1.0), spec["n_x"])
    tg = P.TemporalGrid(spec["horizon"], spec["n_t"])
    assert tg.dt == spec["dt"]
    model = P.make_model(spec["model"], speed=spec.get("speed", 1.0))
    steppers = P.build_steppers(model, sg, tg, n_levels=spec["n_levels"], m=spec["m"],
                                weno_order=spec["weno_order"], stepper=spec["stepper"])
    opts = P.MgritOptions(n_levels=spec["n_levels"], m=spec["m"], cycle=spec["cycle"],
                          relaxation=spec["relaxation"], guess=spec["guess"],
                          max_iters=spec["max_iters"])
    return u0, sg, tg, model, steppers, opts


def _check_history(spec, data, rec, traj):
    name = spec["name"]
    assert rec.diverged_at == spec["diverged_at"], name
    for what in ("residuals", "errors"):
        want = data[f"{name}__{what}"]
        got = getattr(rec, what)
        ok = np.isfinite(want)
        assert np.array_equal(np.isfinite(got), ok), (name, what)
        np.testing.assert_allclose(got[ok], want[ok], rtol=RTOL, atol=0, err_msg=name)
        # exact zeros (sequential exactness) must be exact
        assert np.array_equal(got[ok] == 0.0, want[ok] == 0.0), (name, what)
    if spec["has_traj"] and traj is not None:
        assert np.array_equal(traj, data[name + "__traj"], equal_nan=True), name


def test_every_golden_case(mgrit_golden):
    meta, data = mgrit_golden
    for name, spec in meta.items():
        u0, sg, tg, model, steppers, opts = _problem(spec, data)
        ref = None
        if spec["semantics"] == "harness":
            serial = P.solve_serial(steppers[0], u0, tg, sg, model)
            ref = serial.device_values
        traj, rec = P.mgrit_solve(steppers, u0, tg, sg, opts, reference=ref)
        _check_history(spec, data, rec, traj.values)


def test_drop_in_behind_reference_driver(mgrit_golden):
    """The GPU steppers honour the reference's advance(u)/dt protocol: the
    restated reference driver (oracle/mgrit_oracle.py) run with them
    reproduces the reference histories."""
    meta, data = mgrit_golden
    for name in ("c2_scaled_converging", "fcycle_injection", "order_mix_space_time_up_lf",
                 "single_chunk"):
        spec = meta[name]
        u0, sg, tg, model, steppers, opts = _problem(spec, data)
        ref = None
        if spec["semantics"] == "harness":
            ref = mgrit_oracle.march(steppers[0], u0, spec["n_t"])
        o = mgrit_oracle.Options(n_levels=opts.n_levels, m=opts.m, cycle=opts.cycle,
                                 relaxation=opts.relaxation, guess=opts.guess,
                                 max_iters=opts.max_iters)
        traj, rec = mgrit_oracle.mgrit_solve(steppers, u0, spec["n_t"], tg.dt, o, reference=ref)
        _check_history(spec, data, rec, traj)


def _pair(n_x=32, n_t=64, m=4, L=3, k=2, rk=3, cfl=0.2, seed=7):
    pb = P.Problem(name="ops", n_x=n_x, n_t=n_t, cfl=cfl, n_modes=3, seed=seed,
                   weno_order=(2 * k + 1,), stepper=({1: "fe", 2: "ssprk2", 3: "ssprk3"}[rk],),
                   n_levels=L, m=m)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    gpu = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    ost = [oracle.OracleStepper(k=k, rk_order=rk, dt=tg.dt * m ** l, dx=1.0 / n_x, nthreads=1)
           for l in range(L)]
    cpu = mgrit_oracle.Hierarchy(ost, u0, n_t, tg.dt,
                                 mgrit_oracle.Options(n_levels=L, m=m, relaxation="fcf"))
    return gpu, cpu


def _same(gpu, cpu):
    for l, lv in enumerate(cpu.levels):
        got = gpu.levels[l].u.cpu().numpy()
        assert np.array_equal(got, lv.u, equal_nan=True), l
        if l > 0:
            assert np.array_equal(gpu.levels[l].g.cpu().numpy(), lv.g, equal_nan=True), l


SEQUENCES = [
    ["f0", "c0", "f0", "r0", "f1", "c1", "r1", "cs", "i1", "i0"],
    ["c0", "c0", "f0", "c0", "r0"],              # C-relax from the broadcast state, twice
    ["f0", "c0", "c0", "r0", "cs", "i0"],        # stale F-points (derived from older C)
    ["r0", "r1", "cs", "i1", "i0", "res"],
    ["f0", "res", "c0", "res", "f0", "res"],
]


@pytest.mark.parametrize("seq", SEQUENCES)
def test_level_operations_in_any_order(seq):
    gpu, cpu = _pair()
    for op in seq:
        if op == "res":
            rg, rc = gpu.residual_norm(), cpu.residual_norm()
            assert (np.isnan(rg) and np.isnan(rc)) or abs(rg - rc) <= RTOL * abs(rc)
            continue
        kind, l = op[0], op[1:]
        if op == "cs":
            gpu.coarse_solve(); cpu.coarse_solve()
        elif kind == "f":
            gpu.f_relax(int(l)); cpu.f_relax(int(l))
        elif kind == "c":
            gpu.c_relax(int(l)); cpu.c_relax(int(l))
        elif kind == "r":
            gpu.restrict(int(l)); cpu.restrict(int(l))
        elif kind == "i":
            gpu.interpolate(int(l)); cpu.interpolate(int(l))
        _same(gpu, cpu)


def test_node_zero_never_modified():
    gpu, cpu = _pair()
    u0 = gpu.levels[0].u[0].clone()
    for _ in range(3):
        gpu.run_cycle()
    assert torch.equal(gpu.levels[0].u[0], u0)


def test_c2_full_size_serial_and_first_iteration():
    """BASELINE config 2 at full size: the GPU serial march equals the oracle
    bit for bit; residual row 0 = 2.22175568 and divergence in iteration 1
    (SURVEY.md 8(d))."""
    pb = P.BASELINE_CONFIGS["c2"]
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    sg = pb.space_grid()
    steppers = pb.steppers(tg)
    serial = P.solve_serial(steppers[0], u0, tg, sg, pb.model_obj())
    o = oracle.OracleStepper(k=2, rk_order=3, dt=tg.dt, dx=sg.dx)
    want = mgrit_oracle.march(o, u0, pb.n_t)
    assert np.array_equal(serial.trajectory.values, want)
    opts = P.MgritOptions(n_levels=2, m=4, relaxation="fcf", max_iters=2)
    _, rec = P.mgrit_solve(steppers, u0, tg, sg, opts, reference=serial.device_values,
                           return_trajectory=False)
    assert abs(rec.residuals[0] - 2.22175568) < 5e-8
    assert rec.diverged_at == 1


def test_c3_full_size_row0_and_divergence():
    pb = P.BASELINE_CONFIGS["c3"]
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    opts = P.MgritOptions(n_levels=7, m=4, relaxation="fcf", max_iters=1)
    _, rec = P.mgrit_solve(pb.steppers(tg), u0, tg, pb.space_grid(), opts,
                           return_trajectory=False)
    assert abs(rec.residuals[0] - 6.582632) < 5e-6
    assert rec.diverged_at == 1


def test_large_mesh_mgrit_on_clusters():
    """nx = 8192 (two-CTA clusters for every level operation, cluster-reduced
    residual partials) against the oracle restatement."""
    pb = P.Problem(name="big", n_x=8192, n_t=32, cfl=0.05, n_modes=6, n_levels=3, m=4,
                   relaxation="fcf", max_iters=2)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    steppers = pb.steppers(tg)
    ref = P.serial.march(steppers[0], u0, pb.n_t)
    traj, rec = P.mgrit_solve(steppers, u0, tg, pb.space_grid(), pb.options(), reference=ref)
    ost = [oracle.OracleStepper(k=2, rk_order=3, dt=tg.dt * 4 ** l, dx=1.0 / 8192)
           for l in range(3)]
    oref = mgrit_oracle.march(ost[0], u0, pb.n_t)
    assert np.array_equal(ref.cpu().numpy(), oref)
    otraj, orec = mgrit_oracle.mgrit_solve(ost, u0, pb.n_t, tg.dt,
                                           mgrit_oracle.Options(n_levels=3, m=4,
                                                                relaxation="fcf", max_iters=2),
                                           reference=oref)
    assert np.array_equal(traj.values, otraj)
    np.testing.assert_allclose(rec.residuals, orec.residuals, rtol=1e-10)
    np.testing.assert_allclose(rec.errors, orec.errors, rtol=1e-10)


@pytest.mark.parametrize("relaxation,pieces,n_x", [
    ("fcf", 8, 64), ("fcf", 1, 64), ("f", 3, 64), ("fcf", 1000, 64),
    ("fcf", 0, 2064), ("fcf", 3, 2064)])    # runs of 16 (RK base in global): zero-copy / pieces
def test_relax_to_host_equals_relax_then_fine_values(relaxation, pieces, n_x):
    pb = P.Problem(name="io", n_x=n_x, n_t=256, cfl=0.2, n_modes=3, n_levels=2, m=4,
                   relaxation=relaxation)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    steppers = pb.steppers(tg)
    serial = P.serial.march(steppers[0], u0, pb.n_t)
    c_host = serial[::4, 0].cpu().pin_memory()
    out = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64).pin_memory()
    h = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    h.relax_to_host(c_host, out, pieces=pieces)
    torch.cuda.synchronize()
    g = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    g.load_c_points(c_host)
    g.relax(0)
    assert torch.equal(out, g.fine_values().cpu())
    # the hierarchy state afterwards is the relaxed one
    assert torch.equal(h.fine_values().cpu(), out)


@pytest.mark.parametrize("n_t,kind", [(256, "one zero-copy launch"), (16384, "16 pipelined pieces")])
def test_relax_to_host_default_choice(n_t, kind):
    """pieces=None: below 4096 CF-intervals one launch on the mapped pinned
    buffers, from 4096 on pipelined pieces of 256 intervals; either way the
    result of relax(0) + fine_values()."""
    pb = P.Problem(name="io", n_x=64, n_t=n_t, cfl=0.2, n_modes=3, n_levels=2, m=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    steppers = pb.steppers(tg)
    serial = P.serial.march(steppers[0], u0, pb.n_t)
    c_host = serial[::4, 0].cpu().pin_memory()
    out = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64).pin_memory()
    h = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    h.relax_to_host(c_host, out)
    torch.cuda.synchronize()
    g = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    g.load_c_points(c_host)
    g.relax(0)
    assert torch.equal(out, g.fine_values().cpu()), kind
    assert torch.equal(h.fine_values().cpu(), out), kind


def test_relax_to_host_graph_replay():
    pb = P.Problem(name="io", n_x=64, n_t=256, cfl=0.2, n_modes=3, n_levels=2, m=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    steppers = pb.steppers(tg)
    serial = P.serial.march(steppers[0], u0, pb.n_t)
    c_host = serial[::4, 0].cpu().pin_memory()
    out = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64).pin_memory()
    h = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    g = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    for _ in range(3):          # both buffer parities, captured then replayed
        h.relax_to_host(c_host, out, pieces=4, graph=True)
        torch.cuda.synchronize()
        g.load_c_points(c_host)
        g.relax(0)
        assert torch.equal(out, g.fine_values().cpu())


def test_residual_row_feeds_the_next_c_relaxation():
    """From the second iteration on the finest level's C-relaxation is a
    buffer swap: the residual row before it kept Phi^m(C_j) + 0.0.  Same
    record and trajectory, bit for bit, with fewer launches."""
    pb = P.Problem(name="reuse", n_x=128, n_t=512, cfl=0.05, n_modes=4, n_levels=3, m=4,
                   relaxation="fcf", max_iters=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    out = {}
    for reuse in (True, False):
        P.MgritHierarchy.reuse_residual_for_relaxation = reuse
        try:
            n0 = P._lib.launch_count()
            traj, rec = P.mgrit_solve(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
            out[reuse] = (traj.values, rec.residuals, P._lib.launch_count() - n0)
        finally:
            P.MgritHierarchy.reuse_residual_for_relaxation = True
    assert np.array_equal(out[True][0], out[False][0])
    assert np.array_equal(out[True][1], out[False][1])
    assert out[True][2] == out[False][2] - 3      # iterations 2-4: one launch less each
    # and against the oracle restatement
    ost = [oracle.OracleStepper(k=2, rk_order=3, dt=tg.dt * 4 ** l, dx=1.0 / 128)
           for l in range(3)]
    otraj, orec = mgrit_oracle.mgrit_solve(
        ost, u0, pb.n_t, tg.dt, mgrit_oracle.Options(n_levels=3, m=4, relaxation="fcf",
                                                     max_iters=4))
    assert np.array_equal(out[True][0], otraj)
    np.testing.assert_allclose(out[True][1], orec.residuals, rtol=1e-10)

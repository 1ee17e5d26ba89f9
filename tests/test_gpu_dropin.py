"""Drop-in behind the REAL reference driver: the unmodified reference package
(``mgritlab``, installed into oracle/_ref by ``oracle.install_reference()``
during ``build()``) runs its own ``mgrit_solve`` / ``MgritHierarchy``
(reference mgrit.py:120-340) with the GPU steppers in place of its NumPy
``RungeKuttaStepper`` -- the duck-typed ``advance(u)`` / ``dt`` protocol of
reference tests/test_mgrit.py:34-42.  The records and trajectories must equal
the reference's own run with its own steppers bit for bit."""
import numpy as np
import pytest

import oracle
import paper_2104_09404_b200 as P

pytestmark = pytest.mark.gpu

R = oracle.import_reference()
need_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not installed (build() installs "
                                               "it where /root/reference exists)")

_RK = {"fe": 1, "ssprk2": 2, "ssprk3": 3}

CASES = [
    # (name, n_x, n_t, cfl, n_modes, weno, rk, L, m, cycle, relaxation, guess, iters, harness)
    ("c2_shape_converging", 64, 256, 0.05, 4, 5, "ssprk3", 2, 4, "v", "fcf", "last-step", 6, True),
    ("c3_shape_multilevel", 64, 1024, 0.005, 8, 5, "ssprk3", 4, 4, "v", "fcf", "last-step", 4,
     True),
    ("c4_shape_weno3_f", 64, 512, 0.1, 4, 3, "ssprk2", 3, 2, "v", "f", "last-step", 6, False),
    ("fcycle_injection", 32, 256, 0.1, 4, 3, "ssprk2", 4, 2, "f", "f", "injection", 5, True),
    ("c2_shape_divergent", 64, 256, 0.4, 4, 5, "ssprk3", 2, 4, "v", "fcf", "last-step", 3, True),
    ("single_chunk", 16, 4, 0.3, 2, 5, "ssprk3", 2, 4, "v", "fcf", "last-step", 3, True),
]


def _ref_steppers(sg, tg, weno, rk, L, m):
    model = R.make_model("burgers")
    return [R.RungeKuttaStepper(R.SemiDiscreteOperator(
        model, sg, R.FluxConfig("lf", R.WenoConfig(order=weno))).rhs, tg.dt * m ** l, _RK[rk])
        for l in range(L)]


@need_ref
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_reference_mgrit_solve_with_gpu_steppers(case):
    name, nx, nt, cfl, modes, weno, rk, L, m, cycle, relax, guess, iters, harness = case
    pb = P.Problem(name=name, n_x=nx, n_t=nt, cfl=cfl, n_modes=modes, weno_order=(weno,),
                   stepper=(rk,), n_levels=L, m=m, cycle=cycle, relaxation=relax,
                   guess=guess, max_iters=iters)
    u0 = pb.initial_state()
    tg_p = pb.time_grid(u0)
    sg = R.SpatialGrid(1.0, nx)
    tg = R.TemporalGrid(tg_p.horizon, nt)
    assert tg.dt == tg_p.dt
    opts = R.MgritOptions(n_levels=L, m=m, cycle=cycle, relaxation=relax, guess=guess,
                          max_iters=iters)
    ref_st = _ref_steppers(sg, tg, weno, rk, L, m)
    gpu_st = pb.steppers(tg_p)
    reference = None
    if harness:
        serial = R.solve_serial(ref_st[0], u0, tg, sg, R.make_model("burgers"))
        reference = serial.trajectory.values
        # the GPU serial solve (P.solve_serial) equals the reference's
        g_serial = P.solve_serial(gpu_st[0], u0, tg_p, pb.space_grid(), pb.model_obj())
        assert np.array_equal(g_serial.trajectory.values, reference)
    with np.errstate(all="ignore"):
        want_traj, want = R.mgrit_solve(ref_st, u0, tg, sg, opts, reference=reference)
        got_traj, got = R.mgrit_solve(gpu_st, u0, tg, sg, opts, reference=reference)
    assert got.diverged_at == want.diverged_at, name
    assert np.array_equal(got.errors, want.errors, equal_nan=True), name
    assert np.array_equal(got.residuals, want.residuals, equal_nan=True), name
    assert np.array_equal(got_traj.values, want_traj.values, equal_nan=True), name
    # and the package's own GPU driver reproduces the same record (norms to 1e-10)
    _, own = P.mgrit_solve(gpu_st, u0, tg_p, pb.space_grid(),
                           P.MgritOptions(n_levels=L, m=m, cycle=cycle, relaxation=relax,
                                          guess=guess, max_iters=iters),
                           reference=reference)
    assert own.diverged_at == want.diverged_at
    ok = np.isfinite(want.residuals)
    np.testing.assert_allclose(own.residuals[ok], want.residuals[ok], rtol=1e-10, atol=0)


@need_ref
def test_reference_hierarchy_level_ops_with_gpu_steppers():
    """Level by level: the reference's MgritHierarchy driven by GPU steppers
    holds bit-identical arrays to the one driven by its own steppers."""
    pb = P.Problem(name="ops", n_x=48, n_t=64, cfl=0.2, n_modes=3, n_levels=3, m=4)
    u0 = pb.initial_state()
    tg_p = pb.time_grid(u0)
    sg = R.SpatialGrid(1.0, 48)
    tg = R.TemporalGrid(tg_p.horizon, 64)
    opts = R.MgritOptions(n_levels=3, m=4, relaxation="fcf")
    a = R.MgritHierarchy(_ref_steppers(sg, tg, 5, "ssprk3", 3, 4), u0, tg, sg, opts)
    b = R.MgritHierarchy(pb.steppers(tg_p), u0, tg, sg, opts)
    for op in ("relax0", "restrict0", "relax1", "restrict1", "coarse", "interp1", "interp0",
               "resid", "cycle"):
        for h in (a, b):
            if op == "coarse":
                h.coarse_solve()
            elif op == "resid":
                h._last = h.residual_norm()
            elif op == "cycle":
                h.run_cycle()
            else:
                getattr(h, {"relax": "relax", "restrict": "restrict",
                            "interp": "interpolate"}[op[:-1]])(int(op[-1]))
        for l in range(3):
            assert np.array_equal(a.levels[l].u, b.levels[l].u), (op, l)
            assert np.array_equal(a.levels[l].g, b.levels[l].g), (op, l)
    assert a._last == b._last

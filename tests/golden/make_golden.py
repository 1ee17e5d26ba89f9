"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package (``/root/reference/pkg/src``,
``mgritlab``) read-only, runs its own ``RungeKuttaStepper.advance``,
``SemiDiscreteOperator.rhs`` and ``mgrit_solve`` / ``solve_serial`` on seeded
inputs, and writes

* ``phi_vectors.npz``  -- inputs/outputs of the propagator for every
  (model, WENO degree, RK order, batch regime) combination, including shock
  fields and non-finite cells;
* ``mgrit_cases.npz`` + ``mgrit_cases.json`` -- residual / error histories,
  divergence rows and (small cases) final trajectories of MGRIT runs on
  scaled BASELINE configurations and on checked-in reference configs
  (pkg/configs/high_order_burgers_lf.cfg, order_mix_*_lf.cfg).

The linear-advection model BASELINE config 1 needs is not in the reference
(tests/test_models.py:197-198 rejects it); it is added here as a subclass of
the reference's own ``ConservationModel`` (flux a*u, |lambda| = |a|).  The
GPU box has no /root/reference: the tests read only these committed files.
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, ROOT)

import mgritlab as R  # noqa: E402  (the reference)
from mgritlab.models import ConservationModel  # noqa: E402

import oracle  # noqa: E402
from oracle import mgrit_oracle  # noqa: E402
from paper_2104_09404_b200 import harness as H  # noqa: E402  (IC helpers only)


class RefAdvection(ConservationModel):
    """u_t + a u_x = 0 with the reference model interface (models.py:61-98)."""

    kind = "advection"
    n_components = 1

    def __init__(self, speed=1.0):
        self.speed = float(speed)

    def flux(self, u):
        self._check_shape(u)
        return self.speed * u

    def eigenvalues(self, u):
        self._check_shape(u)
        return np.full(np.moveaxis(u, -2, -1).shape, self.speed)

    def max_abs_speed(self, u):
        self._check_shape(u)
        return np.full(u[..., 0, :].shape, abs(self.speed))


def ref_model(name, speed=1.0):
    return RefAdvection(speed) if name == "advection" else R.make_model(name)


def ref_stepper(model, sg, k, rk, dt, eps=1e-6):
    op = R.SemiDiscreteOperator(model, sg, R.FluxConfig("lf", R.WenoConfig(
        order=2 * k + 1, epsilon=eps)))
    return op, R.RungeKuttaStepper(op.rhs, dt, max(rk, 1))


# ---------------------------------------------------------------------------
# propagator vectors
# ---------------------------------------------------------------------------

def make_fields(rng, shape, kind):
    nx = shape[-1]
    x = (np.arange(nx) + 0.5) / nx
    base = 0.5 + 0.3 * np.sin(2 * np.pi * x) + 0.1 * rng.standard_normal(shape)
    if kind == "shock":
        base = base + np.where(x > 0.4, -0.8, 0.4)
    elif kind == "rough":
        base = rng.standard_normal(shape)
    elif kind == "nan":
        base = base.copy()
        base[..., nx // 3] = np.nan
    elif kind == "inf":
        base = base.copy()
        base[..., 2] = np.inf
    elif kind == "huge":
        base = base.copy()
        base[..., 5] = 1e200
    return np.ascontiguousarray(base, dtype=np.float64)


def phi_vectors():
    rng = np.random.default_rng(20210419)
    out = {}
    index = []
    n = 0
    for model_name in ("burgers", "advection"):
        for k in (0, 1, 2, 3):
            for rk in (0, 1, 2, 3):
                for shape_kind, shape in (("batch", (3, 1, 32)), ("single", (1, 32))):
                    kinds = ["smooth", "shock", "rough"]
                    if rk == 3 and shape_kind == "batch":
                        kinds += ["nan", "inf", "huge"]
                    for fk in kinds:
                        u = make_fields(rng, shape, fk)
                        nx = shape[-1]
                        sg = R.SpatialGrid(1.0, nx)
                        model = ref_model(model_name, speed=-0.75 if model_name == "advection" else 1.0)
                        dt = 0.35 * sg.dx
                        op, st = ref_stepper(model, sg, k, rk, dt)
                        with np.errstate(all="ignore"):
                            y = op.rhs(u) if rk == 0 else st.advance(u)
                        # the oracle must agree bit for bit (NaN-aware)
                        p = oracle.make_params(model=model_name, k=k, rk_order=rk,
                                               dt=dt, dx=sg.dx, speed=model.speed
                                               if model_name == "advection" else 1.0,
                                               regime=oracle.regime_for_shape(shape))
                        mine = oracle.phi_apply(p, u)
                        assert np.array_equal(mine, y, equal_nan=True), (model_name, k, rk, shape, fk)
                        key = f"v{n:04d}"
                        out[key + "_in"] = u
                        out[key + "_out"] = y
                        index.append(dict(key=key, model=model_name, k=k, rk=rk,
                                          shape=list(shape), field=fk, dt=dt, dx=sg.dx,
                                          speed=float(model.speed) if model_name == "advection" else 1.0,
                                          eps=1e-6))
                        n += 1
    # one production-shaped case: WENO5 / SSP-RK3 Burgers, nx = 512
    sg = R.SpatialGrid(1.0, 512)
    u = make_fields(rng, (4, 1, 512), "shock")
    op, st = ref_stepper(R.make_model("burgers"), sg, 2, 3, 0.4 * sg.dx)
    key = f"v{n:04d}"
    out[key + "_in"] = u
    out[key + "_out"] = st.advance(u)
    index.append(dict(key=key, model="burgers", k=2, rk=3, shape=[4, 1, 512],
                      field="shock", dt=0.4 * sg.dx, dx=sg.dx, speed=1.0, eps=1e-6))
    np.savez_compressed(os.path.join(HERE, "phi_vectors.npz"), **out)
    with open(os.path.join(HERE, "phi_vectors.json"), "w") as f:
        json.dump(index, f, indent=0)
    print(f"phi vectors: {len(index)}")


# ---------------------------------------------------------------------------
# MGRIT histories
# ---------------------------------------------------------------------------

_RK = {"fe": 1, "ssprk2": 2, "ssprk3": 3}


def case_ic(spec):
    sg = R.SpatialGrid(spec.get("length", 1.0), spec["n_x"])
    ic = spec["ic"]
    if ic == "fourier":
        return H.fourier_ic(H.SpatialGrid(spec.get("length", 1.0), spec["n_x"]),
                            spec["n_modes"], spec.get("seed", 1234), spec.get("decay", False))
    if ic == "sine":
        return H.sine_ic(H.SpatialGrid(1.0, spec["n_x"]))
    return R.initial_state(ic, sg, spec.get("length", 1.0))


def case_horizon(spec, u0):
    if "horizon" in spec:
        return spec["horizon"]
    sg = R.SpatialGrid(spec.get("length", 1.0), spec["n_x"])
    speed = abs(spec.get("speed", 1.0)) if spec["model"] == "advection" else float(np.max(np.abs(u0)))
    return H.cfl_horizon(spec["n_t"], spec["cfl"], sg.dx, speed)


def run_reference(spec):
    u0 = case_ic(spec)
    sg = R.SpatialGrid(spec.get("length", 1.0), spec["n_x"])
    tg = R.TemporalGrid(case_horizon(spec, u0), spec["n_t"])
    model = ref_model(spec["model"], spec.get("speed", 1.0))
    L, m = spec["n_levels"], spec["m"]
    orders = spec["weno_order"] * (L if len(spec["weno_order"]) == 1 else 1)
    kinds = spec["stepper"] * (L if len(spec["stepper"]) == 1 else 1)
    steppers = []
    for l in range(L):
        op = R.SemiDiscreteOperator(model, sg, R.FluxConfig("lf", R.WenoConfig(
            order=orders[l], epsilon=spec.get("epsilon", 1e-6))))
        steppers.append(R.RungeKuttaStepper(op.rhs, tg.dt * m ** l, _RK[kinds[l]]))
    opts = R.MgritOptions(n_levels=L, m=m, cycle=spec["cycle"],
                          relaxation=spec["relaxation"], guess=spec["guess"],
                          max_iters=spec["max_iters"])
    reference = None
    serial = None
    if spec["semantics"] == "harness":
        serial = R.solve_serial(steppers[0], u0, tg, sg, model)
        reference = serial.trajectory.values
    traj, rec = R.mgrit_solve(steppers, u0, tg, sg, opts, reference=reference)
    # cross-check: the oracle restatement of mgrit.py with oracle steppers
    o_steppers = []
    for l in range(L):
        o_steppers.append(oracle.OracleStepper(
            model=spec["model"], k=(orders[l] - 1) // 2, rk_order=_RK[kinds[l]],
            dt=tg.dt * m ** l, dx=sg.dx, eps=spec.get("epsilon", 1e-6),
            speed=spec.get("speed", 1.0), nthreads=1))
    o_ref = None
    if reference is not None:
        o_ref = mgrit_oracle.march(o_steppers[0], u0, spec["n_t"])
        assert np.array_equal(o_ref, reference)
    o_opts = mgrit_oracle.Options(n_levels=L, m=m, cycle=spec["cycle"],
                                  relaxation=spec["relaxation"], guess=spec["guess"],
                                  max_iters=spec["max_iters"])
    o_traj, o_rec = mgrit_oracle.mgrit_solve(o_steppers, u0, spec["n_t"], tg.dt, o_opts,
                                             reference=o_ref)
    assert o_rec.diverged_at == rec.diverged_at, (spec["name"], o_rec.diverged_at, rec.diverged_at)
    assert np.array_equal(o_traj, traj.values, equal_nan=True), spec["name"]
    ok = np.isfinite(rec.residuals)
    assert np.allclose(o_rec.residuals[ok], rec.residuals[ok], rtol=1e-12, atol=0), spec["name"]
    return u0, tg, rec, traj.values, (serial.trajectory.values if serial else None)


CASES = [
    # BASELINE config 1 at full size (advection, upwind-as-LF, FE, m=8, L=2)
    dict(name="c1_fcf_residual_only", model="advection", speed=1.0, n_x=128, n_t=1024,
         cfl=0.5, ic="sine", weno_order=[1], stepper=["fe"], n_levels=2, m=8, cycle="v",
         relaxation="fcf", guess="last-step", max_iters=66, semantics="residual"),
    dict(name="c1_f_residual_only", model="advection", speed=1.0, n_x=128, n_t=1024,
         cfl=0.5, ic="sine", weno_order=[1], stepper=["fe"], n_levels=2, m=8, cycle="v",
         relaxation="f", guess="last-step", max_iters=130, semantics="residual"),
    dict(name="c1_fcf_harness", model="advection", speed=1.0, n_x=128, n_t=1024,
         cfl=0.5, ic="sine", weno_order=[1], stepper=["fe"], n_levels=2, m=8, cycle="v",
         relaxation="fcf", guess="last-step", max_iters=3, semantics="harness"),
    # BASELINE config 2 shape, scaled (WENO5 / SSP-RK3 Burgers, m=4, L=2, FCF)
    dict(name="c2_scaled", model="burgers", n_x=64, n_t=256, cfl=0.4, ic="fourier",
         n_modes=4, weno_order=[5], stepper=["ssprk3"], n_levels=2, m=4, cycle="v",
         relaxation="fcf", guess="last-step", max_iters=4, semantics="harness"),
    dict(name="c2_scaled_converging", model="burgers", n_x=64, n_t=256, cfl=0.05,
         ic="fourier", n_modes=4, weno_order=[5], stepper=["ssprk3"], n_levels=2, m=4,
         cycle="v", relaxation="fcf", guess="last-step", max_iters=12, semantics="harness"),
    # BASELINE config 3 shape, scaled (multilevel V-cycle, m=4, <=16 coarse steps)
    dict(name="c3_scaled", model="burgers", n_x=64, n_t=1024, cfl=0.005, ic="fourier",
         n_modes=8, weno_order=[5], stepper=["ssprk3"], n_levels=4, m=4, cycle="v",
         relaxation="fcf", guess="last-step", max_iters=8, semantics="harness"),
    dict(name="c3_scaled_divergent", model="burgers", n_x=64, n_t=1024, cfl=0.4,
         ic="fourier", n_modes=8, weno_order=[5], stepper=["ssprk3"], n_levels=4, m=4,
         cycle="v", relaxation="fcf", guess="last-step", max_iters=3, semantics="harness"),
    # BASELINE config 4 style cases (3 levels, F and FCF, WENO1/3/5, RK2/3)
    dict(name="c4_weno5_rk3_fcf", model="burgers", n_x=32, n_t=512, cfl=0.1, ic="fourier",
         n_modes=4, weno_order=[5], stepper=["ssprk3"], n_levels=3, m=2, cycle="v",
         relaxation="fcf", guess="last-step", max_iters=14, semantics="residual"),
    dict(name="c4_weno3_rk2_f", model="burgers", n_x=32, n_t=512, cfl=0.1, ic="fourier",
         n_modes=4, weno_order=[3], stepper=["ssprk2"], n_levels=3, m=2, cycle="v",
         relaxation="f", guess="last-step", max_iters=14, semantics="residual"),
    dict(name="c4_weno1_rk3_f", model="burgers", n_x=32, n_t=512, cfl=0.2, ic="fourier",
         n_modes=4, weno_order=[1], stepper=["ssprk3"], n_levels=3, m=2, cycle="v",
         relaxation="f", guess="last-step", max_iters=10, semantics="residual"),
    # BASELINE config 5 shape, scaled (16 modes a_k/k, m=16)
    dict(name="c5_scaled", model="burgers", n_x=32, n_t=4096, cfl=0.4, ic="fourier",
         n_modes=16, decay=True, weno_order=[5], stepper=["ssprk3"], n_levels=3, m=16,
         cycle="v", relaxation="fcf", guess="last-step", max_iters=2, semantics="residual"),
    # F-cycle + injection guess
    dict(name="fcycle_injection", model="burgers", n_x=32, n_t=256, cfl=0.1, ic="fourier",
         n_modes=4, weno_order=[3], stepper=["ssprk2"], n_levels=4, m=2, cycle="f",
         relaxation="f", guess="injection", max_iters=8, semantics="harness"),
    dict(name="fcycle_fcf_laststep", model="burgers", n_x=32, n_t=256, cfl=0.1, ic="fourier",
         n_modes=4, weno_order=[5], stepper=["ssprk3"], n_levels=3, m=2, cycle="f",
         relaxation="fcf", guess="last-step", max_iters=8, semantics="harness"),
    # single chunk on the finest level (2-lane regime there, general residual path)
    dict(name="single_chunk", model="burgers", n_x=16, n_t=4, cfl=0.3, ic="fourier",
         n_modes=2, weno_order=[5], stepper=["ssprk3"], n_levels=2, m=4, cycle="v",
         relaxation="fcf", guess="last-step", max_iters=3, semantics="harness"),
    # checked-in reference configs (pkg/configs/*.cfg, LF flux, RK steppers)
    *[dict(name=f"high_order_burgers_lf_w{o}", model="burgers", n_x=64, n_t=400,
           horizon=0.5, ic="burgers-43", weno_order=[o], stepper=["ssprk3"], n_levels=3,
           m=2, cycle="v", relaxation="f", guess="last-step", max_iters=10,
           semantics="harness") for o in (1, 3, 5, 7)],
    *[dict(name=f"order_mix_space_lf_{'_'.join(map(str, o))}", model="burgers", n_x=64,
           n_t=400, horizon=0.5, ic="burgers-43", weno_order=list(o), stepper=["ssprk3"],
           n_levels=3, m=2, cycle="v", relaxation="f", guess="last-step", max_iters=10,
           semantics="harness") for o in ((3, 5, 7), (7, 5, 3))],
    dict(name="order_mix_space_time_down_lf", model="burgers", n_x=64, n_t=400,
         horizon=0.5, ic="burgers-43", weno_order=[7, 5, 3],
         stepper=["ssprk3", "ssprk2", "fe"], n_levels=3, m=2, cycle="v", relaxation="f",
         guess="last-step", max_iters=10, semantics="harness"),
    dict(name="order_mix_space_time_up_lf", model="burgers", n_x=64, n_t=400,
         horizon=0.5, ic="burgers-43", weno_order=[3, 5, 7],
         stepper=["fe", "ssprk2", "ssprk3"], n_levels=3, m=2, cycle="v", relaxation="f",
         guess="last-step", max_iters=10, semantics="harness"),
]


def mgrit_cases():
    arrays = {}
    meta = []
    for spec in CASES:
        u0, tg, rec, traj, serial = run_reference(spec)
        key = spec["name"]
        arrays[key + "__u0"] = u0
        arrays[key + "__errors"] = rec.errors
        arrays[key + "__residuals"] = rec.residuals
        if traj.size <= 40000:
            arrays[key + "__traj"] = traj
        m = dict(spec)
        m.update(horizon=tg.horizon, dt=tg.dt, diverged=bool(rec.diverged),
                 diverged_at=rec.diverged_at, has_traj=bool(traj.size <= 40000))
        meta.append(m)
        print(f"{key}: diverged_at={rec.diverged_at} resid[:3]={rec.residuals[:3]}")
    np.savez_compressed(os.path.join(HERE, "mgrit_cases.npz"), **arrays)
    with open(os.path.join(HERE, "mgrit_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


# ---------------------------------------------------------------------------
# one-step Lax-Friedrichs family (stepper.py:85-188) -- SURVEY.md 8(f) rank 1
# ---------------------------------------------------------------------------

def oracle_for(st, dx):
    """Oracle stepper equivalent to a reference stepper object."""
    if isinstance(st, R.ComposedStepper):
        inner = oracle_for(st.inner, dx)
        inner.repeats *= st.repeats
        inner.dt = st.dt
        return inner
    if isinstance(st, (R.MatchedLFFine, R.RediscretizedLF)):
        return oracle.OracleStepper(k=0, rk_order=1, dt=st.dt, dx=dx, scheme=1, nthreads=1)
    if isinstance(st, R.MatchedLFCoarse):
        fdt = st.dt if st.order == 0 else st.dt_fine
        return oracle.OracleStepper(k=0, rk_order=1, dt=st.dt, dx=dx, scheme=2,
                                    lf_order=st.order, m_eff=st.m_effective,
                                    formula_dt=fdt, nthreads=1)
    op = st.rhs.__self__
    return oracle.OracleStepper(model=op.model.kind, k=op.config.weno.degree,
                                rk_order=st.order, dt=st.dt, dx=dx,
                                eps=op.config.weno.epsilon, nthreads=1,
                                scheme=3 if op.config.kind == "roe" else 0)


def lf_vectors():
    rng = np.random.default_rng(7)
    out, index = {}, []
    sg = R.SpatialGrid(1.0, 48)
    model = R.make_model("burgers")
    dt = 0.2 * sg.dx
    op = R.SemiDiscreteOperator(model, sg, R.FluxConfig("lf", R.WenoConfig(5)))
    cases = [("fine", R.MatchedLFFine(model, sg, dt)),
             ("redisc", R.RediscretizedLF(model, sg, 4 * dt))]
    for m_eff in (1, 2, 4, 16):
        for order in (0, 1):
            cases.append((f"matched{order}_m{m_eff}",
                          R.MatchedLFCoarse(model, sg, dt, m_eff, order)))
    cases.append(("composed_fine3", R.ComposedStepper(R.MatchedLFFine(model, sg, dt), 3)))
    for k in (0, 1, 2, 3):
        for rk in (1, 2, 3):
            rop = R.SemiDiscreteOperator(model, sg, R.FluxConfig("roe", R.WenoConfig(2 * k + 1)))
            cases.append((f"roe_k{k}_rk{rk}", R.RungeKuttaStepper(rop.rhs, dt, rk)))
    cases.append(("composed_rk3x4", R.ComposedStepper(R.RungeKuttaStepper(op.rhs, dt, 3), 4)))
    n = 0
    for name, st in cases:
        for shape in ((3, 1, 48), (1, 48)):
            u = make_fields(rng, shape, "shock")
            with np.errstate(all="ignore"):
                y = st.advance(u)
            mine = oracle_for(st, sg.dx).advance(u)
            assert np.array_equal(mine, y, equal_nan=True), name
            key = f"lf{n:03d}"
            out[key + "_in"], out[key + "_out"] = u, y
            meta = dict(key=key, name=name, shape=list(shape), dx=sg.dx, dt_fine=dt)
            if isinstance(st, R.RungeKuttaStepper):
                rop = st.rhs.__self__
                meta.update(kind="roe", k=rop.config.weno.degree, rk=st.order, dt=st.dt)
            elif isinstance(st, R.MatchedLFCoarse):
                meta.update(kind="matched", order=st.order, m_eff=st.m_effective)
            elif isinstance(st, R.ComposedStepper):
                meta.update(kind="composed", repeats=st.repeats,
                            inner="rk3" if isinstance(st.inner, R.RungeKuttaStepper) else "fine")
            else:
                meta.update(kind="onestep", dt=st.dt)
            index.append(meta)
            n += 1
    np.savez_compressed(os.path.join(HERE, "lf_vectors.npz"), **out)
    with open(os.path.join(HERE, "lf_vectors.json"), "w") as f:
        json.dump(index, f, indent=0)
    print(f"lf vectors: {len(index)}")


LF_CONFIGS = [("fine_match_stationary_vcycle.cfg", None),
              ("fine_match_moving_fcycle.cfg", None),
              ("restriction_guess_fcf_relax.cfg", None),
              ("restriction_guess_f_relax.cfg", None),
              ("two_level_exact.cfg", None),
              ("cfl_matched_fe.cfg", None),
              ("fine_match_refinement_vcycle.cfg", 2),
              # Roe flux with entropy fix (flux.py:91-126), SURVEY 8(f) rank 2
              ("high_order_burgers_roe.cfg", None),
              ("order_mix_space_roe.cfg", None),
              ("order_mix_space_time_up_roe.cfg", None),
              ("cfl_weno5_fe_roe.cfg", None),
              ("cfl_weno1_ssprk3_roe.cfg", 3)]


def lf_mgrit_cases():
    arrays, meta = {}, []
    cfg_dir = "/root/reference/pkg/configs"
    for fname, limit in LF_CONFIGS:
        base = R.load_config(os.path.join(cfg_dir, fname))
        cols = [(None, base)] if base.sweep is None else [
            (raw, R.apply_sweep_value(dataclasses.replace(base, sweep=None, sweep_values=()),
                                      base.sweep, raw))
            for raw in base.sweep_values]
        if limit:
            cols = cols[:limit]
        for raw, col in cols:
            res = R.run_experiment(col)
            sg = R.SpatialGrid(col.length, col.n_x)
            tg = R.TemporalGrid(col.horizon, col.n_t)
            u0 = R.initial_state(col.ic, sg, col.length)
            # oracle cross-check with the reference's own steppers mapped
            from mgritlab.harness import build_steppers as ref_build_steppers
            steppers = ref_build_steppers(col, R.make_model(col.problem), sg, tg)
            ost = [oracle_for(st, sg.dx) for st in steppers]
            oref = mgrit_oracle.march(ost[0], u0, col.n_t)
            o_opts = mgrit_oracle.Options(n_levels=col.n_levels, m=col.m, cycle=col.cycle,
                                          relaxation=col.relaxation,
                                          guess=col.restriction_guess,
                                          max_iters=col.max_iters)
            _, orec = mgrit_oracle.mgrit_solve(ost, u0, col.n_t, tg.dt, o_opts, reference=oref)
            assert orec.diverged_at == res.record.diverged_at, fname
            ok = np.isfinite(res.record.errors)
            assert np.allclose(orec.errors[ok], res.record.errors[ok], rtol=1e-12), fname
            name = fname[:-4] + ("" if raw is None else "__" + str(raw).replace(" ", ""))
            arrays[name + "__u0"] = u0
            arrays[name + "__errors"] = res.record.errors
            arrays[name + "__residuals"] = res.record.residuals
            meta.append(dict(name=name, model="burgers", n_x=col.n_x, n_t=col.n_t, flux=col.flux,
                             horizon=col.horizon, dt=tg.dt, length=col.length,
                             stepper=list(col.stepper), weno_order=list(col.weno_order),
                             coarse=col.coarse, n_levels=col.n_levels, m=col.m,
                             cycle=col.cycle, relaxation=col.relaxation,
                             guess=col.restriction_guess, max_iters=col.max_iters,
                             semantics="harness", diverged_at=res.record.diverged_at,
                             has_traj=False))
            print(f"{name}: diverged_at={res.record.diverged_at} err[:3]={res.record.errors[:3]}")
    np.savez_compressed(os.path.join(HERE, "lf_mgrit_cases.npz"), **arrays)
    with open(os.path.join(HERE, "lf_mgrit_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


# ---------------------------------------------------------------------------
# shallow-water system (models.py:130-230, characteristic WENO flux.py:127-161)
# -- SURVEY.md 8(f) rank 4
# ---------------------------------------------------------------------------

def sw_fields(rng, shape, kind):
    nx = shape[-1]
    x = (np.arange(nx) + 0.5) / nx
    lead = shape[:-2]
    u = np.empty(shape)
    u[..., 0, :] = 0.1 + 0.05 * np.sin(2 * np.pi * x) + 0.01 * rng.random(lead + (nx,))
    u[..., 1, :] = 0.02 * rng.standard_normal(lead + (nx,))
    if kind == "bore":
        u[..., 0, :] += np.where(x > 0.5, 0.0, 0.08)
    elif kind == "nan":
        u[..., 1, nx // 3] = np.nan
    elif kind == "dry":      # non-positive depth -> PhysicalStateError
        u[..., 0, 5] = -0.01
    return np.ascontiguousarray(u)


def sw_vectors():
    rng = np.random.default_rng(4)
    out, index = {}, []
    nx = 32
    sg = R.SpatialGrid(1.0, nx)
    model = R.make_model("shallow-water")
    dt = 0.2 * sg.dx
    n = 0
    for flux in ("lf", "roe"):
        for k in (0, 1, 2, 3):
            op = R.SemiDiscreteOperator(model, sg, R.FluxConfig(flux, R.WenoConfig(2 * k + 1)))
            for rk in (0, 1, 2, 3):
                st = R.RungeKuttaStepper(op.rhs, dt, max(rk, 1))
                for shape in ((3, 2, nx), (2, nx)):
                    kinds = ["smooth", "bore"]
                    if rk == 3 and len(shape) == 3:
                        kinds += ["nan", "dry"]
                    for fk in kinds:
                        u = sw_fields(rng, shape, fk)
                        p = oracle.make_params(model="shallow-water", k=k, rk_order=rk,
                                               dt=dt, dx=sg.dx, regime=oracle.SUM_LANE2,
                                               scheme=3 if flux == "roe" else 0)
                        try:
                            with np.errstate(all="ignore"):
                                y = op.rhs(u) if rk == 0 else st.advance(u)
                            raised = False
                        except R.PhysicalStateError:
                            y, raised = np.full_like(u, np.nan), True
                        try:
                            mine = oracle.phi_apply(p, u)
                            assert not raised, (flux, k, rk, fk)
                            assert np.array_equal(mine, y, equal_nan=True), (flux, k, rk, shape, fk)
                        except oracle.PhysicalStateOracleError:
                            assert raised, (flux, k, rk, fk)
                        key = f"sw{n:03d}"
                        out[key + "_in"], out[key + "_out"] = u, y
                        index.append(dict(key=key, flux=flux, k=k, rk=rk, shape=list(shape),
                                          field=fk, dt=dt, dx=sg.dx, gravity=model.gravity,
                                          raises=raised))
                        n += 1
    np.savez_compressed(os.path.join(HERE, "sw_vectors.npz"), **out)
    with open(os.path.join(HERE, "sw_vectors.json"), "w") as f:
        json.dump(index, f, indent=0)
    print(f"sw vectors: {len(index)}")


SW_CONFIGS = ["high_order_shallow_water_lf.cfg", "high_order_shallow_water_roe.cfg"]


def sw_mgrit_cases():
    arrays, meta = {}, []
    cfg_dir = "/root/reference/pkg/configs"
    from mgritlab.harness import build_steppers as ref_build_steppers
    for fname in SW_CONFIGS:
        base = R.load_config(os.path.join(cfg_dir, fname))
        for raw in base.sweep_values:
            col = R.apply_sweep_value(dataclasses.replace(base, sweep=None, sweep_values=()),
                                      base.sweep, raw)
            res = R.run_experiment(col)
            sg = R.SpatialGrid(col.length, col.n_x)
            tg = R.TemporalGrid(col.horizon, col.n_t)
            u0 = R.initial_state(col.ic, sg, col.length)
            steppers = ref_build_steppers(col, R.make_model(col.problem), sg, tg)
            ost = []
            for st in steppers:
                op = st.rhs.__self__
                ost.append(oracle.OracleStepper(
                    model="shallow-water", k=op.config.weno.degree, rk_order=st.order,
                    dt=st.dt, dx=sg.dx, eps=op.config.weno.epsilon, nthreads=1,
                    scheme=3 if op.config.kind == "roe" else 0,
                    gravity=op.model.gravity))
            oref = mgrit_oracle.march(ost[0], u0, col.n_t)
            o_opts = mgrit_oracle.Options(n_levels=col.n_levels, m=col.m, cycle=col.cycle,
                                          relaxation=col.relaxation,
                                          guess=col.restriction_guess,
                                          max_iters=col.max_iters)
            otraj, orec = mgrit_oracle.mgrit_solve(ost, u0, col.n_t, tg.dt, o_opts,
                                                   reference=oref)
            opts = R.MgritOptions(n_levels=col.n_levels, m=col.m, cycle=col.cycle,
                                  relaxation=col.relaxation, guess=col.restriction_guess,
                                  max_iters=col.max_iters)
            traj, rec = R.mgrit_solve(steppers, u0, tg, sg, opts,
                                      reference=res.serial.trajectory.values)
            assert np.array_equal(rec.errors, res.record.errors, equal_nan=True), fname
            assert np.array_equal(oref, res.serial.trajectory.values), fname
            assert orec.diverged_at == res.record.diverged_at, fname
            ok = np.isfinite(res.record.errors)
            assert np.allclose(orec.errors[ok], res.record.errors[ok], rtol=1e-12), fname
            assert np.array_equal(otraj, traj.values, equal_nan=True), fname
            name = fname[:-4] + "__" + str(raw)
            arrays[name + "__u0"] = u0
            arrays[name + "__errors"] = res.record.errors
            arrays[name + "__residuals"] = res.record.residuals
            arrays[name + "__traj"] = traj.values
            meta.append(dict(name=name, model="shallow-water", n_x=col.n_x, n_t=col.n_t,
                             flux=col.flux, horizon=col.horizon, dt=tg.dt, length=col.length,
                             stepper=list(col.stepper), weno_order=list(col.weno_order),
                             coarse=col.coarse, n_levels=col.n_levels, m=col.m,
                             cycle=col.cycle, relaxation=col.relaxation,
                             guess=col.restriction_guess, max_iters=col.max_iters,
                             gravity=R.make_model(col.problem).gravity, ic=col.ic,
                             semantics="harness", diverged_at=res.record.diverged_at,
                             has_traj=True))
            print(f"{name}: diverged_at={res.record.diverged_at} err={res.record.errors}")
    np.savez_compressed(os.path.join(HERE, "sw_mgrit_cases.npz"), **arrays)
    with open(os.path.join(HERE, "sw_mgrit_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


# ---------------------------------------------------------------------------
# PhysicalStateError inside a cycle is recorded as divergence (mgrit.py:
# 316-320); raised by the row-0 residual it propagates (mgrit.py:306-307).
# Shallow-water variants of high_order_shallow_water_*.cfg with a longer
# horizon / fewer steps, found with the reference (coarse CFL too large:
# a depth goes non-positive inside V-cycle 1 or 2).
# ---------------------------------------------------------------------------

SW_DIVERGE = [
    # (name, cfg, horizon, n_t, weno_order, expected outcome in the reference)
    ("sw_psd_lf_T0.75_nt160_w5", "high_order_shallow_water_lf.cfg", 0.75, 160, 5),
    ("sw_psd_lf_T0.75_nt160_w3", "high_order_shallow_water_lf.cfg", 0.75, 160, 3),
    ("sw_psd_lf_T1.0_nt200_w1", "high_order_shallow_water_lf.cfg", 1.0, 200, 1),
    ("sw_psd_roe_T1.0_nt200_w3", "high_order_shallow_water_roe.cfg", 1.0, 200, 3),
    ("sw_psd_lf_T20_nt40_w1_row0", "high_order_shallow_water_lf.cfg", 20.0, 40, 1),
]


def sw_divergence_cases():
    from mgritlab.errors import PhysicalStateError
    from mgritlab.harness import build_steppers as ref_build_steppers
    import mgritlab.mgrit as RM
    arrays, meta = {}, []
    cfg_dir = "/root/reference/pkg/configs"
    for name, fname, horizon, n_t, order in SW_DIVERGE:
        base = R.load_config(os.path.join(cfg_dir, fname))
        col = dataclasses.replace(base, sweep=None, sweep_values=(), weno_order=(order,),
                                  horizon=horizon, n_t=n_t, max_iters=4)
        sg = R.SpatialGrid(col.length, col.n_x)
        tg = R.TemporalGrid(col.horizon, col.n_t)
        model = R.make_model(col.problem)
        u0 = R.initial_state(col.ic, sg, col.length)
        steppers = ref_build_steppers(col, model, sg, tg)
        try:
            reference = R.solve_serial(steppers[0], u0, tg, sg, model).trajectory.values
        except PhysicalStateError:
            reference = None
        opts = R.MgritOptions(n_levels=col.n_levels, m=col.m, cycle=col.cycle,
                              relaxation=col.relaxation, guess=col.restriction_guess,
                              max_iters=col.max_iters)
        # which cycle raised (the record only says diverged_at)
        raised_in_cycle = []
        orig = RM.MgritHierarchy.run_cycle

        def run_cycle(self, _orig=orig):
            try:
                return _orig(self)
            except PhysicalStateError:
                raised_in_cycle.append(True)
                raise
        RM.MgritHierarchy.run_cycle = run_cycle
        try:
            _, rec = R.mgrit_solve(steppers, u0, tg, sg, opts, reference=reference)
            outcome = "recorded"
        except PhysicalStateError:
            rec, outcome = None, "raises"
        finally:
            RM.MgritHierarchy.run_cycle = orig
        ost = [oracle.OracleStepper(model="shallow-water", k=st.rhs.__self__.config.weno.degree,
                                    rk_order=st.order, dt=st.dt, dx=sg.dx, eps=1e-6,
                                    nthreads=1, gravity=model.gravity,
                                    scheme=3 if col.flux == "roe" else 0)
               for st in steppers]
        o_opts = mgrit_oracle.Options(n_levels=col.n_levels, m=col.m, cycle=col.cycle,
                                      relaxation=col.relaxation, guess=col.restriction_guess,
                                      max_iters=col.max_iters)
        if outcome == "raises":
            try:
                mgrit_oracle.mgrit_solve(ost, u0, col.n_t, tg.dt, o_opts)
                raise AssertionError(name + ": oracle did not raise")
            except oracle.PhysicalStateOracleError:
                pass
        else:
            o_ref = None
            if reference is not None:
                o_ref = mgrit_oracle.march(ost[0], u0, col.n_t)
                assert np.array_equal(o_ref, reference), name
            _, orec = mgrit_oracle.mgrit_solve(ost, u0, col.n_t, tg.dt, o_opts,
                                               reference=o_ref)
            assert orec.diverged_at == rec.diverged_at, (name, orec.diverged_at)
            ok = np.isfinite(rec.residuals)
            assert np.allclose(orec.residuals[ok], rec.residuals[ok], rtol=1e-12), name
            arrays[name + "__errors"] = rec.errors
            arrays[name + "__residuals"] = rec.residuals
        arrays[name + "__u0"] = u0
        meta.append(dict(name=name, config=fname, model="shallow-water", n_x=col.n_x,
                         n_t=col.n_t, horizon=col.horizon, length=col.length, flux=col.flux,
                         stepper=list(col.stepper), weno_order=list(col.weno_order),
                         coarse=col.coarse, n_levels=col.n_levels, m=col.m, cycle=col.cycle,
                         relaxation=col.relaxation, guess=col.restriction_guess,
                         max_iters=col.max_iters, gravity=model.gravity, ic=col.ic,
                         has_reference=reference is not None, outcome=outcome,
                         physical_state_error_in_cycle=bool(raised_in_cycle),
                         diverged_at=None if rec is None else rec.diverged_at))
        print(f"{name}: {outcome} diverged_at={None if rec is None else rec.diverged_at}")
    np.savez_compressed(os.path.join(HERE, "sw_diverge_cases.npz"), **arrays)
    with open(os.path.join(HERE, "sw_diverge_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


# ---------------------------------------------------------------------------
# Euler (models.py:214-308) and componentwise systems -- SURVEY.md 8(f) rank 4
#
# The reference takes Euler's left eigenvectors with np.linalg.inv (LAPACK
# via OpenBLAS; models.py:270).  inv3_np below restates that inverse as LU
# with partial pivoting in LAPACK's operation order (the oracle's and the
# kernel's inv3); running the reference with it substituted pins every other
# operation of the Euler path bit for bit, and the unmodified reference's
# outputs give the tolerance check.
# ---------------------------------------------------------------------------

def inv3_np(m):
    a = np.array(m, dtype=float, copy=True)
    shp = a.shape[:-2]
    perm = np.broadcast_to(np.arange(3), shp + (3,)).copy()
    with np.errstate(all="ignore"):
        for j in range(3):
            pv = j + np.argmax(np.abs(a[..., j:, j]), axis=-1)
            idx = pv[..., None, None].repeat(3, -1)
            rj = a[..., j, :].copy()
            a[..., j, :] = np.take_along_axis(a, idx, axis=-2)[..., 0, :]
            np.put_along_axis(a, idx, rj[..., None, :], axis=-2)
            pj = perm[..., j].copy()
            perm[..., j] = np.take_along_axis(perm, pv[..., None], axis=-1)[..., 0]
            np.put_along_axis(perm, pv[..., None], pj[..., None], axis=-1)
            rp = 1.0 / a[..., j, j]
            for i in range(j + 1, 3):
                a[..., i, j] = a[..., i, j] * rp
            for i in range(j + 1, 3):
                for c in range(j + 1, 3):
                    a[..., i, c] = a[..., i, c] - a[..., i, j] * a[..., j, c]
        x = np.empty_like(a)
        for col in range(3):
            b = [(perm[..., i] == col).astype(float) for i in range(3)]
            for kk in range(3):
                nz = b[kk] != 0
                for i in range(kk + 1, 3):
                    b[i] = np.where(nz, b[i] - b[kk] * a[..., i, kk], b[i])
            for kk in (2, 1, 0):
                nz = b[kk] != 0
                b[kk] = np.where(nz, b[kk] / a[..., kk, kk], b[kk])
                for i in range(kk):
                    b[i] = np.where(nz, b[i] - b[kk] * a[..., i, kk], b[i])
            for i in range(3):
                x[..., i, col] = b[i]
    return x


class lu_inverse:
    """Context: the reference's np.linalg.inv replaced by inv3_np."""

    def __enter__(self):
        self.orig = np.linalg.inv
        np.linalg.inv = inv3_np

    def __exit__(self, *exc):
        np.linalg.inv = self.orig


def eu_fields(rng, shape, kind):
    nx = shape[-1]
    x = (np.arange(nx) + 0.5) / nx
    lead = shape[:-2]
    u = np.empty(shape)
    u[..., 0, :] = 1.0 + 0.2 * np.sin(2 * np.pi * x) + 0.05 * rng.random(lead + (nx,))
    u[..., 1, :] = 0.1 * rng.standard_normal(lead + (nx,))
    u[..., 2, :] = 2.0 + 0.3 * rng.random(lead + (nx,))
    if kind == "contact":
        u[..., 0, :] += np.where(x > 0.5, 0.0, 0.6)
    elif kind == "nan":
        u[..., 1, nx // 3] = np.nan
    elif kind == "vacuum":     # non-positive density -> PhysicalStateError
        u[..., 0, 5] = -0.1
    elif kind == "cold":       # non-positive pressure -> PhysicalStateError
        u[..., 2, 7] = 0.0
    return np.ascontiguousarray(u)


def _ref_call(op, st, rk, u):
    try:
        with np.errstate(all="ignore"):
            return (op.rhs(u) if rk == 0 else st.advance(u)), False
    except R.PhysicalStateError:
        return np.full_like(u, np.nan), True


def euler_vectors():
    rng = np.random.default_rng(11)
    out, index = {}, []
    nx = 32
    sg = R.SpatialGrid(1.0, nx)
    dt = 0.2 * sg.dx
    n = 0
    cases = []
    for flux in ("lf", "roe"):
        for k in (0, 1, 2, 3):
            for rk in (0, 1, 2, 3):
                for shape in ((3, 3, nx), (3, nx)):
                    kinds = ["smooth", "contact"]
                    if rk == 3 and len(shape) == 3:
                        kinds += ["nan", "vacuum", "cold"]
                    for fk in kinds:
                        cases.append(("euler", flux, k, rk, shape, fk, True))
    # componentwise reconstruction (WenoConfig.characteristic = False)
    for model in ("euler", "shallow-water"):
        D = 3 if model == "euler" else 2
        for flux in ("lf", "roe"):
            for k in (1, 2, 3):
                for shape in ((3, D, nx), (D, nx)):
                    cases.append((model, flux, k, 3, shape, "smooth", False))
    for model, flux, k, rk, shape, fk, charw in cases:
        m = R.make_model(model)
        op = R.SemiDiscreteOperator(m, sg, R.FluxConfig(flux, R.WenoConfig(
            2 * k + 1, characteristic=charw)))
        st = R.RungeKuttaStepper(op.rhs, dt, max(rk, 1))
        u = eu_fields(rng, shape, fk) if model == "euler" else sw_fields(rng, shape, fk)
        y, raised = _ref_call(op, st, rk, u)
        with lu_inverse():
            y_lu, raised_lu = _ref_call(op, st, rk, u)
        assert raised == raised_lu
        p = oracle.make_params(model=model, k=k, rk_order=rk, dt=dt, dx=sg.dx,
                               regime=oracle.SUM_LANE2, scheme=3 if flux == "roe" else 0,
                               characteristic=charw)
        try:
            mine = oracle.phi_apply(p, u)
            assert not raised, (model, flux, k, rk, fk)
            assert np.array_equal(mine, y_lu, equal_nan=True), (model, flux, k, rk, shape, fk, charw)
        except oracle.PhysicalStateOracleError:
            assert raised, (model, flux, k, rk, fk)
        key = f"eu{n:03d}"
        out[key + "_in"], out[key + "_out"], out[key + "_out_lu"] = u, y, y_lu
        index.append(dict(key=key, model=model, flux=flux, k=k, rk=rk, shape=list(shape),
                          field=fk, characteristic=charw, dt=dt, dx=sg.dx,
                          gamma=R.make_model("euler").gamma, gravity=9.81, raises=raised))
        n += 1
    np.savez_compressed(os.path.join(HERE, "euler_vectors.npz"), **out)
    with open(os.path.join(HERE, "euler_vectors.json"), "w") as f:
        json.dump(index, f, indent=0)
    print(f"euler vectors: {len(index)}")


def euler_configs():
    """high_order_euler_{lf,roe}.cfg: the unmodified reference's tables and
    the LU-inverse reference's error histories (what a bit-exact Euler path
    reproduces up to norm summation order)."""
    out = []
    for name in ("high_order_euler_lf", "high_order_euler_roe"):
        cfg = R.load_config(f"/root/reference/pkg/configs/{name}.cfg")
        res = R.run_sweep(cfg)
        with lu_inverse():
            res_lu = R.run_sweep(cfg)
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            R.emit_csv(res.table, os.path.join(d, "t.csv"))
            text = open(os.path.join(d, "t.csv")).read()
        fields = {k: (list(v) if isinstance(v, tuple) else v)
                  for k, v in dataclasses.asdict(cfg).items()}
        out.append(dict(name=name, config=fields, csv=text, columns=list(res.table.columns),
                        errors_lu=[list(r.record.errors) for r in res_lu.runs],
                        level_dts=[list(r.level_dts) for r in res.runs],
                        level_cfls=[list(r.level_cfls) for r in res.runs],
                        max_speed=[r.serial.max_speed for r in res.runs],
                        diverged_at=[r.record.diverged_at for r in res.runs]))
        print(name, "done")
    with open(os.path.join(HERE, "euler_configs.json"), "w") as f:
        json.dump(out, f, indent=1)


# ---------------------------------------------------------------------------
# the checked-in experiment configs through the reference harness
# (harness.py:369-495) -- SURVEY.md 8(f) rank 3
# ---------------------------------------------------------------------------

def config_tables():
    import glob
    import tempfile
    out = []
    for path in sorted(glob.glob("/root/reference/pkg/configs/*.cfg")):
        cfg = R.load_config(path)
        if cfg.problem == "euler":
            continue      # outside the B200 path
        if cfg.sweep is not None:
            res = R.run_sweep(cfg)
            table, runs = res.table, res.runs
        else:
            run = R.run_experiment(cfg)
            table, runs = R.experiment_table(run), [run]
        with tempfile.TemporaryDirectory() as d:
            csv = os.path.join(d, "t.csv")
            R.emit_csv(table, csv)
            text = open(csv).read()
        fields = {k: (list(v) if isinstance(v, tuple) else v)
                  for k, v in dataclasses.asdict(cfg).items()}
        out.append(dict(name=os.path.basename(path)[:-4], config=fields, csv=text,
                        columns=list(table.columns),
                        level_dts=[list(r.level_dts) for r in runs],
                        level_cfls=[list(r.level_cfls) for r in runs],
                        max_speed=[r.serial.max_speed for r in runs],
                        diverged_at=[r.record.diverged_at for r in runs]))
        print(f"{out[-1]['name']}: {len(runs)} columns")
    with open(os.path.join(HERE, "config_tables.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    import sys as _sys
    which = _sys.argv[1:] or ["phi", "mgrit", "lf", "sw", "euler", "configs"]
    if "euler" in which:
        euler_vectors()
        euler_configs()
    if "configs" in which:
        config_tables()
    if "sw" in which:
        sw_vectors()
        sw_mgrit_cases()
    if "sw" in which or "swdiv" in which:
        sw_divergence_cases()
    if "phi" in which:
        phi_vectors()
    if "mgrit" in which:
        mgrit_cases()
    if "lf" in which:
        lf_vectors()
        lf_mgrit_cases()

"""GPU parity of the shallow-water system kernel:
characteristic WENO with LF / Roe fluxes, bit-identical to the reference
vectors (tests/golden/sw_vectors.*), PhysicalStateError on non-positive depth
(models.py:147-153), and the two checked-in shallow-water configs
(pkg/configs/high_order_shallow_water_{lf,roe}.cfg) through mgrit_solve."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2104_09404_b200 as P

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _stepper(c, nx=None):
    nx = nx or c["shape"][-1]
    sg = P.SpatialGrid(1.0, nx)
    op = P.SemiDiscreteOperator(P.make_model("shallow-water", gravity=c["gravity"]), sg,
                                P.FluxConfig(c["flux"], P.WenoConfig(2 * c["k"] + 1)))
    return op, P.RungeKuttaStepper(op.rhs, c["dt"], max(c["rk"], 1))


def test_sw_vectors_bit_exact(sw_golden):
    index, data = sw_golden
    raised = 0
    for c in index:
        u = data[c["key"] + "_in"]
        op, st = _stepper(c)
        call = (lambda: op.rhs(u)) if c["rk"] == 0 else (lambda: st.advance(u))
        if c["raises"]:
            with pytest.raises(P.PhysicalStateError):
                call()
            raised += 1
            continue
        got = call()
        assert np.array_equal(got, data[c["key"] + "_out"], equal_nan=True), c
    assert raised > 0


@pytest.mark.parametrize("flux", ["lf", "roe"])
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_sw_large_mesh_against_oracle(flux, k):
    """nx = 2048 (the kernel's limit), batch of 5 fields, SSP-RK3."""
    nx = 2048
    rng = np.random.default_rng(100 + k)
    x = (np.arange(nx) + 0.5) / nx
    u = np.empty((5, 2, nx))
    u[:, 0] = 0.1 + 0.04 * np.sin(2 * np.pi * x) + 0.01 * rng.random((5, nx))
    u[:, 1] = 0.02 * rng.standard_normal((5, nx))
    c = dict(flux=flux, k=k, rk=3, dt=0.2 / nx, gravity=9.81, shape=[5, 2, nx])
    _, st = _stepper(c)
    got = st.advance(u)
    p = oracle.make_params(model="shallow-water", k=k, rk_order=3, dt=c["dt"], dx=1.0 / nx,
                           regime=oracle.SUM_LANE2, scheme=3 if flux == "roe" else 0)
    assert np.array_equal(got, oracle.phi_apply(p, u))


def test_sw_composed_and_tensor_io():
    """ComposedStepper over the system kernel (exact coarse operator) with
    CUDA tensors in and out."""
    nx = 64
    c = dict(flux="roe", k=2, rk=3, dt=0.2 / nx, gravity=9.81, shape=[2, nx])
    _, st = _stepper(c)
    comp = P.ComposedStepper(st, 3)
    rng = np.random.default_rng(9)
    u = np.stack([0.1 + 0.01 * rng.random(nx), 0.01 * rng.standard_normal(nx)])
    got = comp.advance(torch.from_numpy(u).cuda())
    assert got.is_cuda and got.shape == (2, nx)
    want = u
    for _ in range(3):
        want = st.advance(want)
    assert np.array_equal(got.cpu().numpy(), want)


def test_sw_rejections():
    sg = P.SpatialGrid(1.0, 4096)
    with pytest.raises(P.ConfigError):
        P.SemiDiscreteOperator(P.make_model("shallow-water"), sg,
                               P.FluxConfig("lf", P.WenoConfig(5)))
    with pytest.raises(P.ConfigError):
        P.make_model("navier-stokes")
    with pytest.raises(P.PhysicalStateError):
        P.make_model("shallow-water", gravity=0.0)


def _sw_cases():
    meta = json.load(open(os.path.join(GOLDEN, "sw_mgrit_cases.json")))
    return [m["name"] for m in meta]


@pytest.mark.parametrize("name", _sw_cases())
def test_sw_reference_configs(sw_mgrit_golden, name):
    meta, data = sw_mgrit_golden
    spec = meta[name]
    sg = P.SpatialGrid(spec["length"], spec["n_x"])
    tg = P.TemporalGrid(spec["horizon"], spec["n_t"])
    model = P.make_model("shallow-water", gravity=spec["gravity"])
    steppers = P.build_steppers(model, sg, tg, n_levels=spec["n_levels"], m=spec["m"],
                                weno_order=spec["weno_order"], stepper=spec["stepper"],
                                flux=spec["flux"])
    u0 = P.harness.named_ic(spec["ic"], sg)
    assert np.array_equal(u0, data[name + "__u0"])
    serial = P.solve_serial(steppers[0], u0, tg, sg, model)
    opts = P.MgritOptions(n_levels=spec["n_levels"], m=spec["m"], cycle=spec["cycle"],
                          relaxation=spec["relaxation"], guess=spec["guess"],
                          max_iters=spec["max_iters"])
    traj, rec = P.mgrit_solve(steppers, u0, tg, sg, opts, reference=serial.device_values)
    assert rec.diverged_at == spec["diverged_at"]
    np.testing.assert_allclose(rec.errors, data[name + "__errors"], rtol=1e-12, atol=0)
    assert np.array_equal(traj.values, data[name + "__traj"])


def test_sw_dry_state_raises_in_solve():
    nx = 64
    sg = P.SpatialGrid(1.0, nx)
    tg = P.TemporalGrid(0.5, 400)
    model = P.make_model("shallow-water")
    steppers = P.build_steppers(model, sg, tg, n_levels=3, m=2, weno_order=(3,),
                                stepper=("ssprk3",), flux="lf")
    u0 = P.harness.named_ic("sw-scaled", sg)
    u0[0, 10] = -0.01
    opts = P.MgritOptions(n_levels=3, m=2, cycle="v", relaxation="f", max_iters=2)
    with pytest.raises(P.PhysicalStateError):
        P.mgrit_solve(steppers, u0, tg, sg, opts)
    with pytest.raises(P.PhysicalStateError):
        P.solve_serial(steppers[0], u0, tg, sg, model)
    # the word is clear again: a good solve runs
    good = P.harness.named_ic("sw-scaled", sg)
    P.mgrit_solve(steppers, good, tg, sg, opts)

"""GPU parity of the fused propagator (through the C ABI) against the
reference's own outputs (golden vectors) and the bit-exact CPU oracle.
Tolerance: bit-exact (NaN-aware) -- the kernels execute the reference's
operation order in IEEE binary64 without FMA contraction."""
import numpy as np
import pytest
import torch

import oracle
import paper_2104_09404_b200 as P

pytestmark = pytest.mark.gpu


def _op(model, k, nx, speed=1.0, eps=1e-6):
    m = P.make_model(model, speed=speed)
    return P.SemiDiscreteOperator(m, P.SpatialGrid(1.0, nx),
                                  P.FluxConfig("lf", P.WenoConfig(2 * k + 1, epsilon=eps)))


def test_phi_matches_reference_golden_vectors(phi_golden):
    index, data = phi_golden
    for c in index:
        u = data[c["key"] + "_in"]
        want = data[c["key"] + "_out"]
        op = _op(c["model"], c["k"], u.shape[-1], c["speed"], c["eps"])
        if c["rk"] == 0:
            got = op.rhs(u)
        else:
            got = P.RungeKuttaStepper(op.rhs, c["dt"], c["rk"]).advance(u)
        assert isinstance(got, np.ndarray) and got.shape == u.shape
        assert np.array_equal(got, want, equal_nan=True), c


@pytest.mark.parametrize("nx", [5, 9, 64, 127, 512, 1000, 2048, 4096])
@pytest.mark.parametrize("k", [0, 1, 2])
@pytest.mark.parametrize("rk", [1, 2, 3])
def test_phi_random_fields_match_oracle(nx, k, rk):
    if nx < 2 * k + 1:
        pytest.skip("mesh too small for the stencil")
    rng = np.random.default_rng(nx * 31 + k * 7 + rk)
    for batch in (1, 3, 17):
        u = rng.standard_normal((batch, 1, nx)) * 0.6 + 0.2
        u[..., nx // 2:] -= 0.9                      # a jump
        dx = 1.0 / nx
        dt = 0.3 * dx
        st = P.RungeKuttaStepper(_op("burgers", k, nx).rhs, dt, rk)
        got = st.advance(u if batch > 1 else u[0])
        p = oracle.make_params(k=k, rk_order=rk, dt=dt, dx=dx,
                               regime=oracle.regime_for_shape(u.shape if batch > 1 else u[0].shape))
        want = oracle.phi_apply(p, u if batch > 1 else u[0])
        assert np.array_equal(got, want), (nx, k, rk, batch)


def test_tensor_in_tensor_out_and_non_pow2_dx():
    nx = 96
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(0.7, nx),
                                P.FluxConfig("lf", P.WenoConfig(5)))
    st = P.RungeKuttaStepper(op.rhs, 0.002, 3)
    rng = np.random.default_rng(3)
    u = rng.standard_normal((5, 1, nx))
    t = torch.from_numpy(u).cuda()
    got = st.advance(t)
    assert torch.is_tensor(got) and got.is_cuda
    want = oracle.phi_apply(oracle.make_params(k=2, rk_order=3, dt=0.002, dx=0.7 / nx), u)
    assert np.array_equal(got.cpu().numpy(), want)
    # the input is never modified (stepper.py:81-82 returns a new array)
    assert np.array_equal(t.cpu().numpy(), u)


def test_advection_upwind_equivalence():
    """First-order LF with |a| = 1 equals upwind to an ulp."""
    nx = 128
    op = _op("advection", 0, nx, speed=1.0)
    st = P.RungeKuttaStepper(op.rhs, 0.5 / nx, 1)
    x = (np.arange(nx) + 0.5) / nx
    u = np.sin(2 * np.pi * x)[None, :]
    got = st.advance(u)
    upwind = u - 0.5 * (u - np.roll(u, 1, axis=-1))
    assert np.max(np.abs(got - upwind)) < 1e-15


@pytest.mark.parametrize("nx,batch", [(8192, 3), (16384, 2), (65536, 2), (1024, 1), (4096, 1)])
def test_cluster_split_fields_match_oracle(nx, batch):
    """Fields above one SM's shared memory (and single-field marches) run on
    a thread-block cluster; results stay bit-exact."""
    rng = np.random.default_rng(nx + batch)
    u = rng.standard_normal((batch, 1, nx)) * 0.5 + 0.4
    u[..., nx // 3: nx // 2] += 0.8
    dx = 1.0 / nx
    dt = 0.4 * dx / np.max(np.abs(u))
    st = P.RungeKuttaStepper(_op("burgers", 2, nx).rhs, dt, 3)
    x = u if batch > 1 else u[0]
    got = st.advance(x)
    want = oracle.phi_apply(oracle.make_params(k=2, rk_order=3, dt=dt, dx=dx,
                                               regime=oracle.regime_for_shape(x.shape)), x)
    assert np.array_equal(got, want), nx


def test_cluster_march_matches_oracle():
    from oracle import mgrit_oracle
    for nx in (512, 2048, 8192):
        rng = np.random.default_rng(nx)
        u0 = 0.5 + 0.3 * np.sin(2 * np.pi * (np.arange(nx) + 0.5) / nx)[None, :]
        u0 = u0 + 0.01 * rng.standard_normal(u0.shape)
        dx = 1.0 / nx
        dt = 0.4 * dx / np.max(np.abs(u0))
        st = P.RungeKuttaStepper(_op("burgers", 2, nx).rhs, dt, 3)
        got = P.serial.march(st, u0, 24).cpu().numpy()
        want = mgrit_oracle.march(oracle.OracleStepper(k=2, rk_order=3, dt=dt, dx=dx), u0, 24)
        assert np.array_equal(got, want), nx

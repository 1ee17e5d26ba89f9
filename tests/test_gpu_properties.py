"""Size-independent properties at the BASELINE configs' own mesh sizes.

Shift equivariance: on a periodic mesh the propagator commutes with cyclic
shifts, Phi(roll(u, s)) = roll(Phi(u), s), and in this implementation BIT FOR
BIT -- every cell is computed by the same operations wherever it sits (the
reference's NumPy arithmetic has the same property), and the global alpha is a
max.  A shift moves every cell to another thread, run position, CTA slab and
halo, so the test exercises every boundary of every kernel against its
interior: the batched sweeps (runs of 8), the LL groups (slabs of 4096 cells
over global memory), the fused FCF launch (runs of 4 / 8 / 16) and the cluster
march.
"""
import numpy as np
import pytest
import torch

import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import device as dev
from paper_2104_09404_b200._lib import G_ZERO, SUM_SEQ, TAIL_PHI

pytestmark = pytest.mark.gpu


def _stepper(nx, order=5, rk=3):
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, nx),
                                P.FluxConfig("lf", P.WenoConfig(order)))
    return P.RungeKuttaStepper(op.rhs, 0.3 / nx, rk)


def _field(nx, seed):
    rng = np.random.default_rng(seed)
    x = (np.arange(nx) + 0.5) / nx
    u = 0.4 + 0.3 * np.sin(2 * np.pi * x) + 0.1 * np.sin(2 * np.pi * 7 * x + 1.0)
    u = u + 0.02 * rng.standard_normal(nx)
    u[nx // 3: nx // 2] += 0.5
    return u


SHIFTS = (1, 2, 7, 8, 9, 15, 16, 17, 255, 4095, 4096, 4099)


@pytest.mark.parametrize("nx,order,rk", [(4096, 5, 3), (65536, 5, 3), (32768, 5, 3),
                                         (1024, 3, 2), (1024, 1, 1), (512, 5, 3)])
def test_batched_sweep_is_shift_equivariant(nx, order, rk):
    st = _stepper(nx, order, rk)
    u = _field(nx, nx + order)
    shifts = [s % nx for s in SHIFTS]
    x = torch.from_numpy(np.stack([u] + [np.roll(u, s) for s in shifts])).cuda()
    n = x.shape[0]
    steps = 2
    store = torch.empty(n, steps, nx, dtype=torch.float64, device="cuda")
    tail = torch.empty(n, nx, dtype=torch.float64, device="cuda")
    dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=n, start=x, start_stride=nx, n_steps=steps,
              g_mode=G_ZERO, store=store, st_cs=steps * nx, st_ss=nx, tail=TAIL_PHI,
              tail_regime=SUM_SEQ, tail_g_mode=G_ZERO, tail_out=tail, to_s=nx)
    assert torch.isfinite(tail).all()
    for i, s in enumerate(shifts, start=1):
        assert torch.equal(tail[i], torch.roll(tail[0], s)), (nx, s)
        assert torch.equal(store[i], torch.roll(store[0], s, dims=-1)), (nx, s)


@pytest.mark.parametrize("nx", [512, 1024, 4096])
def test_fused_fcf_relaxation_is_shift_equivariant(nx):
    """Interval j holds the field shifted by SHIFTS[j]: every chain of the
    fused launch (runs of 4, 8 and 16 cells for the three meshes) must return
    the shifted copy of chain 0's states."""
    shifts = [0] + [s % nx for s in SHIFTS]
    m = 4
    nc = len(shifts)
    pb = P.Problem(name="shift", n_x=nx, n_t=m * nc, cfl=0.2, n_modes=3, n_levels=2, m=m)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    u = _field(nx, 3)
    c = np.stack([np.roll(u, s) for s in shifts] + [u])
    h = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    h.load_c_points(c)
    assert h._fcf_workspace() is not None
    out = h.relax_fine_values().reshape(nc * m + 1, nx)
    # chain j: F-steps and C-step from C_j  ->  new C_{j+1}; then interval
    # j+1's final F-steps from it.  Rows j*m + 1 .. j*m + m - 1 are interval
    # j's final F-points (from NEW C_j), row (j+1)*m the new C_{j+1}.
    newc = out[m::m]                                   # new C_1 .. C_nc
    for j, s in enumerate(shifts):
        assert torch.equal(newc[j], torch.roll(newc[0], s)), (nx, "C", s)
    # final F-points of interval j (j >= 1) start from new C_j = roll(new C_1, shift_{j-1})
    for j in range(2, nc):
        s = shifts[j - 1]
        for i in range(1, m):
            assert torch.equal(out[j * m + i], torch.roll(out[m + i], s)), (nx, "F", s, i)


@pytest.mark.parametrize("nx,order", [(512, 5), (4096, 5), (1024, 3), (256, 1)])
def test_cluster_march_is_shift_equivariant(nx, order):
    st = _stepper(nx, order, 3)
    u = _field(nx, 11)
    base = P.serial.march(st, u[None], 6)[:, 0]
    for s in (1, 33, nx // 16 + 1, nx - 1):
        got = P.serial.march(st, np.roll(u, s)[None], 6)[:, 0]
        assert torch.equal(got, torch.roll(base, s, dims=-1)), (nx, s)

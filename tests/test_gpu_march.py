"""GPU parity of march_kernel -- the one-barrier-per-stage sequential march
of one field over a thread-block cluster (coarse solve mgrit.py:219-226,
serial solve serial.py:40-61) -- against the two-barrier Field path and the
CPU oracle's march, bit for bit (NaN-aware), for every cluster size it
accepts, first order, WENO3 and WENO5, both summation regimes, every Runge-Kutta order
and every g mode.
The path is selected per call through MGP_MARCH2 / MGP_MARCH_CS (read by
the library at each launch)."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import device as dev
from paper_2104_09404_b200._lib import G_ARRAY, G_NONE, G_ZERO, SUM_LANE2, SUM_SEQ

pytestmark = pytest.mark.gpu


def _phi(nx, rk, regime, cfl=0.3, order=5):
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, nx),
                                P.FluxConfig("lf", P.WenoConfig(order)))
    st = P.RungeKuttaStepper(op.rhs, cfl / nx, rk)
    return st.phi_struct(regime), cfl / nx


def _field(nx, seed, bad=None):
    rng = np.random.default_rng(seed)
    x = (np.arange(nx) + 0.5) / nx
    u = 0.5 + 0.25 * np.sin(2 * np.pi * x + rng.uniform(0, 2 * np.pi)) \
        + 0.1 * rng.standard_normal(nx)
    u[nx // 3: nx // 2] -= 0.7                     # a jump
    if bad == "nan":
        u[nx // 5] = np.nan
    elif bad == "inf":
        u[nx - 2] = np.inf
    elif bad == "huge":
        u[nx // 4] = 1e200                          # slow-path divisions
    return u


def _run(phi, u0, n, g_mode, g, env):
    nx = u0.shape[-1]
    traj = torch.empty(n + 1, nx, dtype=torch.float64, device="cuda")
    traj[0] = torch.from_numpy(u0).cuda()
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        dev.sweep(phi, n_chunks=1, start=traj, start_stride=0, n_steps=n, g_mode=g_mode,
                  g=None if g is None else g[1], g_ss=nx, store=traj[1], st_ss=nx,
                  what="march")
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return traj.cpu().numpy()


def _np(x):
    return x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def _bits_equal(a, b):
    return np.array_equal(a.view(np.int64), b.view(np.int64)) or \
        np.array_equal(a, b, equal_nan=True)


CASES = [(nx, cs) for nx in (32, 64, 128, 512, 1024, 4096) for cs in (2, 4, 8, 16)
         if nx % cs == 0 and 8 <= nx // cs <= 256]


@pytest.mark.parametrize("nx,cs", CASES)
@pytest.mark.parametrize("rk", [1, 2, 3])
@pytest.mark.parametrize("regime", [SUM_LANE2, SUM_SEQ])
@pytest.mark.parametrize("order", [1, 3, 5])
def test_march_kernel_equals_field_path(nx, cs, rk, regime, order):
    phi, _ = _phi(nx, rk, regime, order=order)
    u0 = _field(nx, nx + cs + rk)
    n = 24
    got = _run(phi, u0, n, G_NONE, None, {"MGP_MARCH_CS": str(cs)})
    want = _run(phi, u0, n, G_NONE, None, {"MGP_MARCH2": "0"})
    assert _bits_equal(got, want)


@pytest.mark.parametrize("g_mode", [G_NONE, G_ZERO, G_ARRAY])
@pytest.mark.parametrize("bad", [None, "nan", "inf", "huge"])
@pytest.mark.parametrize("order", [1, 3, 5])
def test_march_kernel_equals_oracle(g_mode, bad, order):
    nx, n, rk = 128, 16, 3
    k = order // 2
    phi, dt = _phi(nx, rk, SUM_LANE2, order=order)
    u0 = _field(nx, 7, bad)
    g = None
    if g_mode == G_ARRAY:
        g = np.random.default_rng(1).standard_normal((n + 1, nx)) * 1e-3
    gd = None if g is None else torch.from_numpy(g).cuda()
    for cs in (2, 4, 8, 16):
        got = _run(phi, u0, n, g_mode, gd, {"MGP_MARCH_CS": str(cs)})
        want = np.empty((n + 1, nx))
        want[0] = u0
        p = oracle.make_params(k=k, rk_order=rk, dt=dt, dx=1.0 / nx, regime=SUM_LANE2)
        gz = None
        if g_mode == G_ARRAY:
            gz = g.copy()
        elif g_mode == G_ZERO:
            gz = np.zeros((n + 1, nx))
        oracle.march(p, want, gz, n)
        assert _bits_equal(got, want), (cs, g_mode, bad)


def test_march_kernel_drives_coarse_solve_and_serial():
    """The public paths that use it: solve_serial and the coarsest level's
    solve give the same trajectories with march_kernel and the Field path."""
    pb = P.Problem(name="march", n_x=256, n_t=256, cfl=0.2, n_modes=4, n_levels=2, m=4,
                   max_iters=2)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    res = []
    for env in ({"MGP_MARCH_CS": "4"}, {"MGP_MARCH2": "0"}):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            s = P.serial.march(st[0], u0, pb.n_t)
            traj, rec = P.mgrit_solve(st, u0, tg, pb.space_grid(), pb.options())
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        res.append((_np(s), _np(traj.values), _np(rec.residuals)))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2], equal_nan=True)

"""Split meshes (N_x > 4096) swept by groups of co-resident CTAs that exchange
halo cells, edge states and alpha through global memory ("LL" mode of
csrc/mgrit_phi.cu, the default for batched sweeps) -- against the
thread-block-cluster path (MGP_LL=0) and against the oracle.

Every mgp_sweep feature that crosses the group is covered: chained steps with
and without a g array (fused commit and copy-loop paths), every tail
(Phi, FAS restriction, residual), partial sums over the ranks, the error and
non-finite counters, more chunks than groups, fewer chunks than groups,
non-finite fields.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import device as dev
from paper_2104_09404_b200._lib import (G_ARRAY, G_NONE, G_ZERO, GUESS_LAST_STEP, SUM_SEQ,
                                        TAIL_NONE, TAIL_PHI, TAIL_RESID, TAIL_RESTRICT)

pytestmark = pytest.mark.gpu


def _stepper(nx, dt_scale=1.0):
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, nx),
                                P.FluxConfig("lf", P.WenoConfig(5)))
    return P.RungeKuttaStepper(op.rhs, dt_scale * 0.3 / nx, 3)


def _fields(nx, n, seed):
    rng = np.random.default_rng(seed)
    x = (np.arange(nx) + 0.5) / nx
    u = 0.5 + 0.3 * np.sin(2 * np.pi * (x[None, :] + rng.random((n, 1))))
    u = u + 0.02 * rng.standard_normal((n, nx))
    u[:, nx // 3: nx // 2] += 0.4          # jumps: every nonlinear weight regime
    return torch.from_numpy(u).cuda()


class _Env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _both(fn):
    """Run fn() on the LL path (default) and on the cluster path."""
    with _Env(MGP_LL=1):
        a = fn()
    with _Env(MGP_LL=0):
        b = fn()
    torch.cuda.synchronize()
    return a, b


@pytest.mark.parametrize("nx,nc", [(8192, 3), (8192, 90), (16384, 5), (32768, 4),
                                   (65536, 2), (65536, 20),
                                   (8200, 5),      # 4 slabs of 2050 cells: partial last run
                                   (12300, 3)])    # 4 slabs of 3075 cells (odd)
@pytest.mark.parametrize("g_mode", [G_ZERO, G_ARRAY])
def test_chained_steps_and_tail_phi(nx, nc, g_mode):
    st = _stepper(nx)
    phi = st.phi_struct(SUM_SEQ)
    x = _fields(nx, nc, nx + nc)
    steps = 3
    g = 1e-3 * _fields(nx, nc * steps, 7).reshape(nc, steps, nx) if g_mode == G_ARRAY else None

    def run():
        store = torch.full((nc, steps, nx), np.nan, dtype=torch.float64, device="cuda")
        tail = torch.full((nc, nx), np.nan, dtype=torch.float64, device="cuda")
        dev.sweep(phi, n_chunks=nc, start=x, start_stride=nx, n_steps=steps, g_mode=g_mode,
                  g=g, g_cs=steps * nx, g_ss=nx, store=store, st_cs=steps * nx, st_ss=nx,
                  tail=TAIL_PHI, tail_regime=SUM_SEQ, tail_g_mode=G_ZERO, tail_out=tail, to_s=nx)
        return store, tail

    (s1, t1), (s0, t0) = _both(run)
    assert torch.isfinite(s1).all() and torch.isfinite(t1).all()
    assert torch.equal(s1, s0) and torch.equal(t1, t0)


@pytest.mark.parametrize("nx,nc", [(8192, 4), (16384, 3), (8200, 3), (12300, 2)])
def test_against_oracle(nx, nc):
    st = _stepper(nx)
    x = _fields(nx, nc, 11)
    steps = 2
    store = torch.empty(nc, steps, nx, dtype=torch.float64, device="cuda")
    dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=nx, n_steps=steps,
              g_mode=G_NONE, store=store, st_cs=steps * nx, st_ss=nx)
    p = oracle.make_params(k=2, rk_order=3, dt=st.dt, dx=1.0 / nx, regime=oracle.SUM_SEQ)
    u = x.cpu().numpy()[:, None, :]
    for s in range(steps):
        u = oracle.phi_apply(p, u)
        assert np.array_equal(store[:, s].cpu().numpy(), u[:, 0]), (nx, s)


@pytest.mark.parametrize("nx,nc", [(8192, 5), (65536, 11)])
def test_residual_tail_partials_and_counters(nx, nc):
    st = _stepper(nx)
    phi = st.phi_struct(SUM_SEQ)
    x = _fields(nx, nc + 1, 3)
    ref = _fields(nx, (nc + 1) * 3, 5).reshape(nc + 1, 3, nx)
    tgt = x[1:] + 1e-4

    def run():
        part = torch.full((3 * nc,), np.nan, dtype=torch.float64, device="cuda")
        dev.sweep(phi, n_chunks=nc, start=x, start_stride=nx, n_steps=2, g_mode=G_ZERO,
                  tail=TAIL_RESID, tail_regime=SUM_SEQ, tail_g_mode=G_ZERO, aux=tgt, aux_s=nx,
                  ref=ref, ref_cs=3 * nx, ref_ss=nx, ref_last_next=1, count_nonfinite=1,
                  partials=part)
        return part

    a, b = _both(run)
    assert torch.isfinite(a).all()
    assert torch.equal(a, b)


@pytest.mark.parametrize("nx,nc", [(8192, 300), (65536, 40)])
def test_partials_without_any_step(nx, nc):
    """The monitor's pass over stored states: no step, no tail, only the
    error / non-finite partial sums -- chunks without an alpha exchange, so
    the partial-sum exchange must pace itself."""
    st = _stepper(nx)
    x = _fields(nx, 3, 9)
    ref = _fields(nx, nc, 10)

    def run():
        part = torch.full((3 * nc,), np.nan, dtype=torch.float64, device="cuda")
        dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=0, ref=ref,
                  ref_cs=nx, count_nonfinite=1, partials=part)
        return part

    a, b = _both(run)
    assert torch.isfinite(a).all() and torch.equal(a, b)
    want = ((x[0][None, :] - ref) ** 2).sum(dim=1)
    np.testing.assert_allclose(a.reshape(nc, 3)[:, 1].cpu().numpy(), want.cpu().numpy(),
                               rtol=1e-12)


@pytest.mark.parametrize("nx,nc", [(8192, 6), (32768, 10)])
def test_restriction_tail(nx, nc):
    fine, coarse = _stepper(nx), _stepper(nx, 4.0)
    x = _fields(nx, nc, 21)
    phi_f = _fields(nx, nc, 22)
    g_f = 1e-3 * _fields(nx, nc, 23)
    inj = _fields(nx, nc, 24)

    def run():
        gc = torch.full((nc, nx), np.nan, dtype=torch.float64, device="cuda")
        uc = torch.full((nc, nx), np.nan, dtype=torch.float64, device="cuda")
        dev.sweep(coarse.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=nx,
                  tail=TAIL_RESTRICT, tail_regime=SUM_SEQ, tail_g_mode=G_ARRAY, tail_g=g_f,
                  tg_s=nx, guess=GUESS_LAST_STEP, aux=phi_f, aux_s=nx, aux2=inj, aux2_s=nx,
                  tail_out=gc, to_s=nx, tail_out2=uc, to2_s=nx)
        return gc, uc

    (g1, u1), (g0, u0) = _both(run)
    assert torch.isfinite(g1).all()
    assert torch.equal(g1, g0) and torch.equal(u1, u0)
    del fine


def test_nonfinite_fields_propagate_identically():
    nx, nc = 16384, 6
    st = _stepper(nx)
    x = _fields(nx, nc, 31)
    x[1, 5] = float("nan")          # next to a slab edge
    x[2, nx // 4] = float("inf")    # on a slab edge (4 slabs of 4096)
    x[3, nx - 1] = 1e200            # overflow in the smoothness products
    x[4, 0] = float("nan")

    def run():
        store = torch.zeros(nc, 2, nx, dtype=torch.float64, device="cuda")
        dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=nx, n_steps=2,
                  g_mode=G_ZERO, store=store, st_cs=2 * nx, st_ss=nx)
        return store

    a, b = _both(run)
    assert torch.equal(torch.isnan(a), torch.isnan(b))
    assert torch.equal(torch.nan_to_num(a, nan=0.0, posinf=1.0, neginf=-1.0),
                       torch.nan_to_num(b, nan=0.0, posinf=1.0, neginf=-1.0))
    assert torch.isnan(a[1]).all() and torch.isfinite(a[0]).all() and torch.isfinite(a[5]).all()
    want = oracle.phi_apply(
        oracle.make_params(k=2, rk_order=3, dt=st.dt, dx=1.0 / nx, regime=oracle.SUM_SEQ),
        x.cpu().numpy()[:, None, :])
    got = a[:, 0].cpu().numpy()
    assert np.array_equal(np.isnan(got), np.isnan(want[:, 0]))
    ok = np.isfinite(want[:, 0])
    assert np.array_equal(got[ok], want[:, 0][ok])


def test_repeated_launches_reuse_the_mailbox():
    """Tags restart at 1 with every launch: the mailbox is cleared in stream
    order, so back-to-back launches on one stream cannot see stale words."""
    nx, nc = 8192, 7
    st = _stepper(nx)
    phi = st.phi_struct(SUM_SEQ)
    x = _fields(nx, nc, 41)
    outs = []
    for _ in range(4):
        out = torch.empty(nc, nx, dtype=torch.float64, device="cuda")
        dev.sweep(phi, n_chunks=nc, start=x, start_stride=nx, n_steps=1, g_mode=G_ZERO,
                  tail=TAIL_PHI, tail_regime=SUM_SEQ, tail_g_mode=G_ZERO, tail_out=out, to_s=nx)
        outs.append(out)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    assert TAIL_NONE == 0

"""Small invocations of every round-2 kernel path (fused FCF launch with runs
of 4 / 8 / 16 cells, batched sweeps with every epilogue, LL groups, the
st.async march, a 3-level solve) -- sized for compute-sanitizer
(`compute-sanitizer --tool racecheck python tools/sanitize_probe.py`).  The
tool is closed on this round's GPU pool, so the paths are validated by the
bit-exact parity tests instead; the script stays as the entry point."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import device as dev  # noqa: E402
from paper_2104_09404_b200._lib import G_ARRAY, G_NONE, G_ZERO, SUM_SEQ, TAIL_PHI, TAIL_RESID  # noqa: E402

which = sys.argv[1:] or ["fcf", "fcf16", "sweep", "ll", "march", "mgrit"]


def stepper(nx):
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, nx),
                                P.FluxConfig("lf", P.WenoConfig(5)))
    return P.RungeKuttaStepper(op.rhs, 0.3 / nx, 3)


def fields(nx, n):
    x = (np.arange(nx) + 0.5) / nx
    u = 0.5 + 0.3 * np.sin(2 * np.pi * (x[None, :] + 0.1 * np.arange(n)[:, None]))
    return torch.from_numpy(u).cuda()


def fcf(nx, nt):
    pb = P.Problem(name="s", n_x=nx, n_t=nt, cfl=0.2, n_modes=3, n_levels=2, m=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    h = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    h.load_c_points(np.stack([np.roll(u0[0], j) for j in range(nt // 4 + 1)]))
    out = h.relax_fine_values()
    torch.cuda.synchronize()
    return float(out.sum())


if "fcf" in which:
    print("fcf runs of 4/8:", fcf(64, 64), fcf(1024, 16))
if "fcf16" in which:
    print("fcf runs of 16 (RK base in global):", fcf(2064, 16))
if "sweep" in which:
    nx, nc = 256, 5
    st = stepper(nx)
    x = fields(nx, nc + 1)
    part = torch.zeros(3 * nc, dtype=torch.float64, device="cuda")
    g = 1e-3 * fields(nx, nc * 2).reshape(nc, 2, nx)
    store = torch.zeros(nc, 2, nx, dtype=torch.float64, device="cuda")
    for gm, garr in ((G_ZERO, None), (G_ARRAY, g)):
        dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=nx, n_steps=2,
                  g_mode=gm, g=garr, g_cs=2 * nx, g_ss=nx, store=store, st_cs=2 * nx, st_ss=nx,
                  tail=TAIL_RESID, tail_regime=SUM_SEQ, tail_g_mode=G_ZERO, aux=x[1], aux_s=nx,
                  count_nonfinite=1, partials=part)
    torch.cuda.synchronize()
    print("sweep:", float(part.sum()))
if "ll" in which:
    nx, nc = 8192, 3
    st = stepper(nx)
    x = fields(nx, nc + 1)
    part = torch.zeros(3 * nc, dtype=torch.float64, device="cuda")
    out = torch.zeros(nc, nx, dtype=torch.float64, device="cuda")
    dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=nx, n_steps=2,
              g_mode=G_ZERO, tail=TAIL_RESID, tail_regime=SUM_SEQ, tail_g_mode=G_ZERO,
              aux=x[1], aux_s=nx, count_nonfinite=1, partials=part)
    dev.sweep(st.phi_struct(SUM_SEQ), n_chunks=nc, start=x, start_stride=nx, n_steps=1,
              g_mode=G_NONE, tail=TAIL_PHI, tail_regime=SUM_SEQ, tail_g_mode=G_ZERO,
              tail_out=out, to_s=nx)
    torch.cuda.synchronize()
    print("ll groups:", float(part.sum()), float(out.sum()))
if "march" in which:
    for nx in (128, 512):
        st = stepper(nx)
        u0 = fields(nx, 1).cpu().numpy()
        print("march", nx, float(P.serial.march(st, u0, 12).sum()))
if "mgrit" in which:
    pb = P.Problem(name="s", n_x=64, n_t=64, cfl=0.1, n_modes=3, n_levels=3, m=4, max_iters=2)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    _, rec = P.mgrit_solve(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    print("mgrit residuals", rec.residuals.tolist())

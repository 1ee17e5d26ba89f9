"""GPU parity of the fused finest-level FCF relaxation (mgp_relax_fcf): one
launch, single steps handed out to persistent CTAs from a ticket counter
with the field travelling through an L2 ring between steps, must
equal the two-sweep path (fused F+C sweep, then the F-relaxation storing
every F-point) bit for bit -- new C-points, trajectory, node 0 -- for chain
splits of every shape (shares shorter and longer than a chain, fewer
intervals than CTAs), every WENO degree and coarsening factor."""
import pytest
import torch

import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import device as dev

pytestmark = pytest.mark.gpu


def _pair(pb, segment=0, split=0):
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    steppers = pb.steppers(tg)
    serial = P.serial.march(steppers[0], u0, pb.n_t)
    c = serial[::pb.m, 0]
    fused = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    plain = P.MgritHierarchy(steppers, u0, tg, pb.space_grid(), pb.options())
    plain._fcf_ws = None                     # force the two-sweep path
    fused._fcf_segment = segment
    fused._fcf_split = split
    for h in (fused, plain):
        h.load_c_points(c)
    assert fused._fcf_workspace() is not None
    return fused, plain


CASES = [
    # n_x, n_t, m, weno_order, stepper: shares cut chains at varying points
    (512, 4096, 4, 5, "ssprk3"),      # BASELINE config 2 (1024 intervals > CTAs)
    (64, 4096, 4, 5, "ssprk3"),       # many small fields: high occupancy
    (256, 2048, 8, 5, "ssprk3"),      # long chains (15 steps)
    (128, 512, 2, 5, "ssprk3"),
    (96, 120, 4, 5, "ssprk3"),        # 30 intervals: one chain per CTA
    (128, 1024, 4, 3, "ssprk2"),      # WENO3
    (128, 1024, 4, 1, "fe"),          # first order
    (128, 1024, 4, 7, "ssprk3"),      # WENO7
    (1024, 2048, 4, 5, "ssprk3"),     # runs of 8 cells per thread
    (4096, 2400, 4, 5, "ssprk3"),     # runs of 16, RK base in global memory, 2 CTAs/SM;
                                      # 600 intervals > 296 CTA slots
    (2064, 256, 4, 5, "ssprk2"),      # runs of 16, 129 threads' worth of cells, SSP-RK2
    (3000, 64, 2, 5, "ssprk3"),       # above 2048 but not a multiple of 16: runs of 8
]


@pytest.mark.parametrize("segment", [0, 1, 2, 3])
@pytest.mark.parametrize("nx,nt,m,order,stepper", CASES)
def test_relax_fine_values_equals_two_sweeps(nx, nt, m, order, stepper, segment):
    pb = P.Problem(name="fcf", n_x=nx, n_t=nt, m=m, cfl=0.3, n_modes=4,
                   weno_order=(order,), stepper=(stepper,))
    fused, plain = _pair(pb, segment)
    for _ in range(2):                       # both ping-pong parities
        got = fused.relax_fine_values()
        plain.relax(0)
        want = plain.fine_values()
        assert torch.equal(got, want)
        assert torch.equal(fused.c_points(), plain.c_points())


@pytest.mark.parametrize("split", [-1, 0, 1, 7, 600, 100000])
@pytest.mark.parametrize("nx,nt,m,order,stepper", [CASES[0], CASES[1], CASES[2], CASES[4]])
def test_split_plan_equals_two_sweeps(nx, nt, m, order, stepper, split):
    """Split plan: the first chains run F + C only and queue their final
    F-steps, taken later in completion order from the new C-point in cd."""
    pb = P.Problem(name="fcf-split", n_x=nx, n_t=nt, m=m, cfl=0.3, n_modes=4,
                   weno_order=(order,), stepper=(stepper,))
    fused, plain = _pair(pb, 0, split)
    for _ in range(3):                       # both parities, workspace reused
        got = fused.relax_fine_values()
        plain.relax(0)
        assert torch.equal(got, plain.fine_values())
        assert torch.equal(fused.c_points(), plain.c_points())


def test_c_relax_fused_equals_sweep():
    pb = P.BASELINE_CONFIGS["c2"]
    fused, plain = _pair(pb)
    for h in (fused, plain):
        h.f_relax(0)
        h.c_relax(0)
    assert torch.equal(fused.c_points(), plain.c_points())
    assert torch.equal(fused.fine_values(), plain.fine_values())


def test_fused_mgrit_iterations_match_unfused():
    pb = P.Problem(name="fcf-it", n_x=128, n_t=1024, cfl=0.1, n_modes=3, n_levels=3,
                   m=2, max_iters=4)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    a = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    b = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    b._fcf_ws = None
    for _ in range(4):
        a.run_cycle()
        b.run_cycle()
        assert torch.equal(a.fine_values(), b.fine_values())
        assert a.residual_norm() == b.residual_norm()


@pytest.mark.parametrize("segment", [0, 1, 2])
def test_relax_to_host_pieces_fused(segment):
    pb = P.BASELINE_CONFIGS["c2"]
    fused, plain = _pair(pb, segment)
    c_host = fused.c_points().reshape(-1, pb.n_x).cpu().pin_memory()
    out = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64).pin_memory()
    for pieces in (1, 2, 3, 1, 0):          # workspace reused; 0 = zero-copy launch
        fused.relax_to_host(c_host, out, pieces=pieces)
        torch.cuda.synchronize()
        plain.load_c_points(c_host)
        plain.relax(0)
        assert torch.equal(out, plain.fine_values().cpu()), pieces


def test_workspace_query_and_rejections():
    pb = P.BASELINE_CONFIGS["c2"]
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    phi = pb.steppers(tg)[0].phi_struct(dev.regime_for_batch(1024))
    nb = dev.fcf_workspace_bytes(phi, 1024, 4)
    # four counters, then a tag / queue word and a hand-over row per resident
    # CTA slot (the layout does not depend on the interval count)
    slots = (nb - 32) // (8 + 512 * 8)
    assert nb == 32 + slots * (8 + 512 * 8) and 148 <= slots <= 148 * 16
    assert dev.fcf_workspace_bytes(phi, 8, 4) == nb
    lane2 = pb.steppers(tg)[0].phi_struct(dev.regime_for_batch(1))
    assert dev.fcf_workspace_bytes(lane2, 1024, 4) == 0     # single-field regime
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    c = torch.zeros(1025, 512, dtype=torch.float64, device="cuda")
    with pytest.raises(P.ConfigError):
        dev.relax_fcf(phi, n_chunks=1024, m=4, g_mode=1, cs=c, cd=c.clone(),
                      workspace=ws[: nb // 2])           # workspace too small


@pytest.mark.parametrize("window", ["1", "7", "192", "0"])
def test_relax_to_host_zero_copy_ordered_loads(window):
    """Zero-copy input: chain-start loads in ticket order with a bounded
    window (MGP_FCF_ORDERED, read per launch; 0 = unordered) -- any window,
    split or segment plan, gives the plain relaxation bit for bit."""
    import os
    pb = P.BASELINE_CONFIGS["c2"]
    for segment, split in ((0, 0), (0, -1), (2, 0)):
        fused, plain = _pair(pb, segment, split)
        c_host = fused.c_points().reshape(-1, pb.n_x).cpu().pin_memory()
        out = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64).pin_memory()
        old = os.environ.get("MGP_FCF_ORDERED")
        os.environ["MGP_FCF_ORDERED"] = window
        try:
            for _ in range(2):                  # workspace counters reset by the launch
                fused.relax_to_host(c_host, out, pieces=0)
                torch.cuda.synchronize()
                plain.load_c_points(c_host)
                plain.relax(0)
                assert torch.equal(out, plain.fine_values().cpu()), (window, segment, split)
                c_host = fused.c_points().reshape(-1, pb.n_x).cpu().pin_memory()
        finally:
            if old is None:
                os.environ.pop("MGP_FCF_ORDERED", None)
            else:
                os.environ["MGP_FCF_ORDERED"] = old

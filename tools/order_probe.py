"""Throughput of the fused FCF relaxation (F-points stored) for the lower-order
schemes of BASELINE config 4 at scale (N_x = 1024, 32768 intervals): point-
updates/s, and the HBM write rate of the stored trajectory (8 B per
point-update) against the measured copy bandwidth."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
FLOPS = {(5, "ssprk3"): 735, (3, "ssprk3"): 297, (3, "ssprk2"): 197, (1, "ssprk3"): 45,
         (1, "ssprk2"): 29, (1, "fe"): 13}
for order, stp in [(5, "ssprk3"), (3, "ssprk3"), (3, "ssprk2"), (1, "ssprk3"), (1, "ssprk2"), (1, "fe")]:
    nx, nt = 1024, 131072
    pb = P.BASELINE_CONFIGS["c4"].scaled(name="p", n_x=nx, n_t=nt, n_levels=2, m=4,
                                         weno_order=(order,), stepper=(stp,), relaxation="fcf")
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    nc = nt // pb.m
    c = np.stack([np.roll(u0[0], j % nx) for j in range(nc + 1)])
    h = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    out = torch.empty(nt + 1, nx, dtype=torch.float64, device="cuda")
    h.load_c_points(c)
    h.relax_fine_values(out=out)
    ts = []
    for _ in range(5):
        h.load_c_points(c)
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        h.relax_fine_values(out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    pts = 7 * nc * nx
    gbs = (8 * (nt + 1) * nx + 16 * (nc + 1) * nx) / ms / 1e6
    print(f"WENO{order} {stp:7s}: {ms:7.3f} ms  {pts / ms / 1e6:7.2f} G pt-upd/s  "
          f"{pts / ms / 1e6 * FLOPS[(order, stp)] / 1e3:6.2f} TFLOP/s  HBM {gbs:7.1f} GB/s", flush=True)
    del h, out

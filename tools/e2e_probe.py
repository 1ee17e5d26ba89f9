"""Where does the zero-copy e2e step lose time?  One fused FCF launch with
the C-points read from host (mapped) or device memory and the trajectory
written to host (mapped) or device memory, CUDA events, C2."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import device as dev  # noqa: E402
from paper_2104_09404_b200._lib import G_ZERO  # noqa: E402

pb = P.BASELINE_CONFIGS["c2"]
u0 = pb.initial_state()
tg = pb.time_grid(u0)
st = pb.steppers(tg)
h = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
serial = P.serial.march(st[0], u0, pb.n_t)
nc, nx, m = pb.n_t // pb.m, pb.n_x, pb.m
c_dev = serial[::m, 0].reshape(nc + 1, nx).contiguous()
c_host = c_dev.cpu().pin_memory()
t_dev = torch.empty(pb.n_t + 1, nx, dtype=torch.float64, device="cuda")
t_host = torch.empty(pb.n_t + 1, nx, dtype=torch.float64).pin_memory()
cd = torch.empty_like(c_dev)
ws = h._fcf_workspace()
phi = h._phi(0, dev.regime_for_batch(nc))
flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
for name, cs, tr in (("in host, out host", c_host, t_host), ("in host, out dev", c_host, t_dev),
                     ("in dev, out host", c_dev, t_dev if False else t_host),
                     ("in dev, out dev", c_dev, t_dev)):
    ts = []
    for it in range(25):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dev.relax_fcf(phi, n_chunks=nc, m=m, g_mode=G_ZERO, cs=cs, cd=cd, workspace=ws,
                      split=0, fstore=tr[1], f_cs=m * nx, f_ss=nx, cstore=tr, cst_s=m * nx)
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{name:20s} median {ts[len(ts)//2]*1e3:7.1f} us  min {ts[0]*1e3:7.1f} us")

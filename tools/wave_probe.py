"""Throughput of the fused F+C sweep (C2 shape: nx 512, m 4, WENO5/RK3) as a
function of the number of chunks -- exposes the partial-wave tail."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import device as dev  # noqa: E402
from paper_2104_09404_b200._lib import G_ZERO, TAIL_PHI  # noqa: E402


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return sorted(out)[len(out) // 2]


pb = P.BASELINE_CONFIGS["c2"]
u0 = pb.initial_state()
tg = pb.time_grid(u0)
st = pb.steppers(tg)[0]
nx, m = pb.n_x, pb.m
res = {}
for nc in [int(x) for x in (sys.argv[1:] or "148 296 444 592 740 888 1024 1184 1776 2368 4736".split())]:
    x = dev.to_device(u0).reshape(nx).expand(nc, nx).contiguous()
    y = torch.empty_like(x)
    phi = st.phi_struct(0)
    f = lambda: dev.sweep(phi, n_chunks=nc, start=x, start_stride=nx, n_steps=m - 1,
                          g_mode=G_ZERO, tail=TAIL_PHI, tail_out=y, to_s=nx)
    ms = timed(f)
    res[nc] = round(m * nc * nx / ms / 1e6, 3)
print(os.environ.get("MGP_RUN", "auto"), json.dumps(res))

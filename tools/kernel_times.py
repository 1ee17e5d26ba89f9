"""Ad-hoc kernel timings on finite data (CUDA events): relaxation sweeps and
the sequential coarse solve, for the BASELINE shapes."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import device as dev  # noqa: E402
from paper_2104_09404_b200._lib import G_NONE, G_ZERO, TAIL_PHI  # noqa: E402


def timed(fn, reps=5):
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
    return min(out)


res = {}
for name in sys.argv[1:] or ["c2", "c3"]:
    pb = P.BASELINE_CONFIGS[name]
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)[0]
    nx, m = pb.n_x, pb.m
    nc = pb.n_t // m
    if os.environ.get("MGP_KT_MAXCHUNKS"):   # C5: a bounded sample of the intervals
        nc = min(nc, int(os.environ["MGP_KT_MAXCHUNKS"]))
    x = dev.to_device(u0).reshape(nx).expand(nc, nx).contiguous()
    y = torch.empty_like(x)
    phi = st.phi_struct(0)
    f = lambda: dev.sweep(phi, n_chunks=nc, start=x, start_stride=nx, n_steps=m - 1,
                          g_mode=G_ZERO, tail=TAIL_PHI, tail_out=y, to_s=nx)
    ms = timed(f)
    pts = m * nc * nx
    res[name + "_fused_fc_ms"] = ms
    res[name + "_fused_fc_gpts"] = pts / ms / 1e6
    if os.environ.get("MGP_KT_NOMARCH"):
        continue
    # sequential march: n steps of the finest propagator from u0 (finite)
    n = min(1024, pb.n_t)
    traj = torch.empty(n + 1, nx, dtype=torch.float64, device="cuda")
    traj[0] = x[0]
    g = lambda: dev.sweep(st.phi_struct(1), n_chunks=1, start=traj, start_stride=0,
                          n_steps=n, g_mode=G_NONE, store=traj[1], st_ss=nx)
    ms = timed(g, 3)
    res[name + f"_march{n}_ms"] = ms
    res[name + "_march_us_per_step"] = 1e3 * ms / n
print(json.dumps(res, indent=1))

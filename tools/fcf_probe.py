"""Fused FCF relaxation (mgp_relax_fcf, relax_fine_values) vs the two-sweep
path, C2 shape (nx 512, m 4, WENO5/RK3) at several interval counts."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402


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


base = P.BASELINE_CONFIGS["c2"]
res = {}
for nc in [int(x) for x in (sys.argv[1:] or "296 592 1024 1184 2368 4736".split())]:
    pb = base.scaled(n_t=nc * base.m)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    c = torch.from_numpy(u0).cuda().reshape(1, -1).expand(nc + 1, -1).contiguous()
    out = torch.empty(pb.n_t + 1, pb.n_x, dtype=torch.float64, device="cuda")
    row = {}
    variants = [("fused_whole", True, -1), ("fused_split_auto", True, 0),
                ("two_sweeps", False, 0)]
    for sp in os.environ.get("MGP_PROBE_SPLITS", "").split():
        variants.append((f"split_{sp}", True, int(sp)))
    for name, fused, split in variants:
        h = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
        h._fcf_split = split
        if not fused:
            h._fcf_ws = None
        h.load_c_points(c)
        ms = timed(lambda: h.relax_fine_values(out=out))
        row[name] = round((2 * pb.m - 1) * nc * pb.n_x / ms / 1e6, 3)
    res[nc] = row
print(json.dumps(res))

"""Timings of the bench step (one fused FCF relaxation of the finest level,
F-points stored: MgritHierarchy.relax_fine_values) for library variants.

    MGP_LIB_PATH=tools/exp/X.so python tools/fcf_times.py c2 c3

Input: C-point j = the config's initial state rolled by j cells (finite,
non-trivial, no serial march needed, so experiment builds that lack the
march kernels work).  Prints per config the median ms over 7 steps (L2
flushed before each), G point-updates/s and a digest of the output
trajectory, so variants can be checked bit for bit against the release
library."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests"))
import paper_2104_09404_b200 as P  # noqa: E402
from fixture_hash import canonical_hash  # noqa: E402

res = {"lib": os.environ.get("MGP_LIB_PATH", "release")}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for name in sys.argv[1:] or ["c2", "c3"]:
    pb = P.BASELINE_CONFIGS[name]
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    nc = pb.n_t // pb.m
    c = np.stack([np.roll(u0[0], j % pb.n_x) for j in range(nc + 1)])
    h = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    out = torch.empty(pb.n_t + 1, pb.n_x, dtype=torch.float64, device="cuda")
    h.load_c_points(c)
    h.relax_fine_values(out=out)
    digest = canonical_hash(out.cpu().numpy())
    ts = []
    for _ in range(7):
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
    pts = (2 * pb.m - 1) * nc * pb.n_x
    res[name] = {"ms": ms, "gpts": pts / ms / 1e6, "frac": pts / ms / 1e6 * 735 / 18540,
                 "digest": digest[:16]}
print(json.dumps(res))

"""Per-CTA start/end/SM of one fused FCF launch (experiment build with
-DMGP_CTA_TIMES), C2 shape at the given interval count."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import _lib  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 4736
base = P.BASELINE_CONFIGS["c2"]
pb = base.scaled(n_t=nc * base.m)
u0 = pb.initial_state()
tg = pb.time_grid(u0)
st = pb.steppers(tg)
c = torch.from_numpy(u0).cuda().reshape(1, -1).expand(nc + 1, -1).contiguous()
out = torch.empty(pb.n_t + 1, pb.n_x, dtype=torch.float64, device="cuda")
h = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
h.load_c_points(c)
for _ in range(3):
    h.relax_fine_values(out=out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 2048))()
_lib.load().mgp_debug_cta_times(buf)
a = np.array(buf, dtype=np.float64).reshape(-1, 3)
G = int(h._fcf_ws.numel() // (2 * pb.n_x * 8 + 4))
a = a[:G]
t0 = a[:, 0].min()
s_, e_ = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
print(f"G={G} start us: min {s_.min():.1f} max {s_.max():.1f} p50 {np.median(s_):.1f}")
print(f"end us: min {e_.min():.1f} max {e_.max():.1f} p50 {np.median(e_):.1f}")
print("duration us percentiles 0/10/50/90/100:",
      np.percentile(e_ - s_, [0, 10, 50, 90, 100]).round(1).tolist())
sm = a[:, 2].astype(int)
cnt = np.bincount(sm, minlength=148)
print("CTAs per SM histogram:", np.bincount(cnt).tolist())
print("start-time histogram (us bins of 2):", np.histogram(s_, bins=10)[0].tolist(),
      np.histogram(s_, bins=10)[1].round(1).tolist())

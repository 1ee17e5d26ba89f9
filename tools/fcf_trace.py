"""Per-ticket timeline of one fused FCF launch (experiment build with
-DMGP_FCF_TRACE): CTA work spans, per-SM busy slots over time, the tail."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import _lib  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
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
buf = (ctypes.c_ulonglong * (4 * 8192))()
_lib.load().mgp_debug_fcf_trace(buf)
a = np.array(buf, dtype=np.uint64).reshape(-1, 4)
a = a[a[:, 1] > 0]
t0 = a[:, 0].min()
s_ = (a[:, 0] - t0).astype(float) / 1e3
e_ = (a[:, 1] - t0).astype(float) / 1e3
cta = a[:, 2].astype(int)
sm = (a[:, 3] & 0xffffffff).astype(int)
steps = (a[:, 3] >> 32).astype(int)
dur = (e_ - s_) / steps
print(f"tickets {len(a)} makespan {e_.max():.1f} us; per-step us p10/50/90: "
      f"{np.percentile(dur, [10, 50, 90]).round(2).tolist()}")
ends = np.zeros(cta.max() + 1)
for k in range(len(a)):
    ends[cta[k]] = max(ends[cta[k]], e_[k])
print("CTA finish us percentiles 0/10/50/90/100:", np.percentile(ends, [0, 10, 50, 90, 100]).round(1).tolist())
busy = [(np.sum((s_ <= t) & (e_ > t))) for t in np.linspace(0, e_.max(), 21)]
print("busy CTAs over time:", busy)
tick_gap = []
for q in range(cta.max() + 1):
    idx = np.where(cta == q)[0]
    idx = idx[np.argsort(s_[idx])]
    for x, y in zip(idx[:-1], idx[1:]):
        tick_gap.append(s_[y] - e_[x])
print("gap between a CTA's units us p50/p90:", np.percentile(tick_gap, [50, 90]).round(2).tolist() if tick_gap else None)

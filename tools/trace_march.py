import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import _lib, device as dev
from paper_2104_09404_b200._lib import G_NONE
pb = P.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
u0 = pb.initial_state(); tg = pb.time_grid(u0); st = pb.steppers(tg)[0]
nx = pb.n_x
traj = torch.empty(33, nx, dtype=torch.float64, device="cuda"); traj[0] = dev.to_device(u0)[0]
f = lambda: dev.sweep(st.phi_struct(1), n_chunks=1, start=traj, start_stride=0, n_steps=32, g_mode=G_NONE, store=traj[1], st_ss=nx)
f(); torch.cuda.synchronize()
lib = _lib.load(); lib.mgp_trace_read.restype = ctypes.c_int
buf = (ctypes.c_longlong * 8192)()
lib.mgp_trace_read(buf, 8192)
f(); torch.cuda.synchronize()
n = lib.mgp_trace_read(buf, 8192)
ev = [(buf[2*i], buf[2*i+1]) for i in range(n)]
# durations between consecutive tags
from collections import defaultdict
acc = defaultdict(list)
for (t0, a), (t1, b) in zip(ev, ev[1:]):
    acc[f"{t0}->{t1}"].append(b - a)
print(json.dumps({k: [len(v), sum(v)/len(v)] for k, v in acc.items()}, indent=0))
print("total ns", ev[-1][1] - ev[0][1], "events", n)

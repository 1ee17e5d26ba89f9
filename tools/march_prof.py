"""Per-phase cycle totals of march_kernel (thread 0 of CTA 0, clock64), from
an MGP_TRACE build: recon, warp max + slot stores, cluster barrier, alpha,
flux/update, __syncthreads."""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import _lib, device as dev
from paper_2104_09404_b200._lib import G_NONE
pb = P.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
u0 = pb.initial_state(); tg = pb.time_grid(u0); st = pb.steppers(tg)[0]
nx = pb.n_x; n = 256
traj = torch.empty(n + 1, nx, dtype=torch.float64, device="cuda"); traj[0] = dev.to_device(u0)[0]
f = lambda: dev.sweep(st.phi_struct(1), n_chunks=1, start=traj, start_stride=0, n_steps=n,
                      g_mode=G_NONE, store=traj[1], st_ss=nx)
f(); f(); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * 8192)()
lib.mgp_trace_read(buf, 8192)
names = ["recon", "umax+slots", "barrier", "alpha", "update", "syncthreads"]
tot = {names[buf[2 * i]]: round(buf[2 * i + 1] / (3 * n), 1) for i in range(6)}
tot["sum_per_stage"] = round(sum(v for v in tot.values()), 1)
print(json.dumps(tot))

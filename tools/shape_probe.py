"""Throughput of the fused FCF relaxation (F-points stored) by mesh size at
equal total work: how many CTAs share an SM (profiles/r02_fcf_u0g.txt)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2104_09404_b200 as P
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for nx, nt in [(512, 262144), (1024, 131072), (2048, 65536), (4096, 32768), (4096, 65536)]:
    pb = P.BASELINE_CONFIGS["c3"].scaled(name="p", n_x=nx, n_t=nt, n_levels=2)
    u0 = pb.initial_state(); tg = pb.time_grid(u0)
    nc = nt // pb.m
    c = np.stack([np.roll(u0[0], j % nx) for j in range(nc + 1)])
    h = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    out = torch.empty(nt + 1, nx, dtype=torch.float64, device="cuda")
    h.load_c_points(c); h.relax_fine_values(out=out)
    ts = []
    for _ in range(5):
        h.load_c_points(c); flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); h.relax_fine_values(out=out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts)); pts = 7 * nc * nx
    print(f"nx {nx:5d} intervals {nc:6d}: {ms:8.3f} ms  {pts / ms / 1e6:6.2f} G  frac {pts / ms / 1e6 * 735 / 18540:.3f}", flush=True)
    del h, out

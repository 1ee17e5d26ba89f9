"""Per-launch breakdown of one MGRIT iteration (V-cycle + residual row) of a
BASELINE config: which sweep / fused launch takes how long (CUDA events)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import device as dev
import paper_2104_09404_b200.mgrit as M
log = []
def wrap(name, orig):
    def traced(phi, **kw):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); r = orig(phi, **kw); b.record()
        log.append((name, kw.get('what'), kw['n_chunks'], kw.get('n_steps', kw.get('m', 0)), kw.get('tail', 0), kw.get('g_mode', 0), a, b))
        return r
    return traced
M.dev.sweep = wrap('sweep', dev.sweep)
M.dev.relax_fcf = wrap('fcf', dev.relax_fcf)
pb = P.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
u0 = pb.initial_state(); tg = pb.time_grid(u0)
for rep in range(2):
    h = P.MgritHierarchy(pb.steppers(tg), u0, tg, pb.space_grid(), pb.options())
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.run_cycle(); mon = h.monitor()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
tot = 0
for name, what, nc, ns, tail, g, a, b in log:
    ms = a.elapsed_time(b); tot += ms
    if ms > 0.2: print(f"{name:5s} {what:18s} nc={nc:6d} steps={ns:2d} tail={tail} g={g} {ms:8.3f} ms")
print("sum of launches", tot, "wall", wall * 1e3, "n launches", len(log))

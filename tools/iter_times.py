"""Whole MGRIT iteration timings (V-cycle + residual row) and finest-level
relaxation throughput on finite data, for the BASELINE configs."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


out = {}
for name in sys.argv[1:]:
    pb = P.BASELINE_CONFIGS[name]
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = pb.steppers(tg)
    t0 = time.perf_counter()
    h = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    m0 = h.monitor()
    torch.cuda.synchronize()
    # warm-up on a throwaway hierarchy: first-call costs (function attributes,
    # the FCF workspace) stay out of the timed relaxation
    w = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    w.relax(0)
    if pb.n_x * pb.n_t <= 1 << 26:   # small configs: also load every kernel of a cycle
        w.run_cycle()
        w.monitor()
    torch.cuda.synchronize()
    del w
    # relaxation on finite data (the initial iterate): FCF on level 0
    a, b = ev(), ev()
    a.record()
    h.relax(0)
    b.record()
    torch.cuda.synchronize()
    relax_ms = a.elapsed_time(b)
    n1 = pb.n_t // pb.m
    pts = pb.m * n1 * pb.n_x          # fused F+C work actually executed
    # one full iteration from the initial iterate (one hierarchy alive: its
    # peak is the config's memory footprint)
    del h
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    h = P.MgritHierarchy(st, u0, tg, pb.space_grid(), pb.options())
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    h.run_cycle()
    mon = h.monitor()
    b.record()
    torch.cuda.synchronize()
    out[name] = {"setup_s": setup, "row0_residual": m0.residual,
                 "relax0_ms": relax_ms, "relax0_gpts": pts / relax_ms / 1e6,
                 "iteration_ms": a.elapsed_time(b), "residual_after_it1": mon.residual,
                 "nonfinite_after_it1": mon.nonfinite,
                 "mem_gb": torch.cuda.max_memory_allocated() / 1e9}
    del h
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
print(json.dumps(out, indent=1))

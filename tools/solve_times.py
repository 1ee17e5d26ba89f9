"""Whole-solve timing: a converging config-3-shaped problem (N_x = 4096,
N_t = 16384, CFL 0.05, two levels, 5 iterations), with and without the reuse of the
residual row's propagator chain for the next C-relaxation."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402

pb = P.BASELINE_CONFIGS["c3"].scaled(name="solve", n_t=16384, cfl=0.05, n_levels=2, max_iters=5)
u0 = pb.initial_state()
tg = pb.time_grid(u0)
for reuse in (True, False, True, False):
    P.MgritHierarchy.reuse_residual_for_relaxation = reuse
    st = pb.steppers(tg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rec = P.mgrit_solve(st, u0, tg, pb.space_grid(), pb.options(), return_trajectory=False)
    torch.cuda.synchronize()
    print(f"reuse={reuse}: {1e3 * (time.perf_counter() - t0):8.2f} ms  residuals "
          f"{[float(f'{r:.3e}') for r in rec.residuals]}", flush=True)

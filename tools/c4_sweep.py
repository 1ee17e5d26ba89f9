"""BASELINE config 4 at full size on one B200: Burgers, Nx = 1024,
Nt = 16384, 3-level MGRIT, grid over CFL x m x scheme x integrator x
relaxation (192 cases); per case: iterations to residual < 1e-10 (within 10
iterations), divergence iteration, wall time per iteration and fine
point-updates/s of the whole solve (reference-equivalent propagator
applications x Nx / solve time)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402


def phi_per_iteration(pb):
    c = pb.relaxation_phi_per_iteration()
    return c["relaxation"] + c["restriction"] + c["coarse"] + c["residual"]


def main():
    cases = P.c4_grid()
    if len(sys.argv) > 1:
        cases = cases[: int(sys.argv[1])]
    out = []
    t_all = time.perf_counter()
    for pb in cases:
        pb = pb.scaled(residual_tol=1e-10, max_iters=10)
        u0 = pb.initial_state()
        tg = pb.time_grid(u0)
        st = pb.steppers(tg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rec = P.mgrit_solve(st, u0, tg, pb.space_grid(), pb.options(),
                               return_trajectory=False, residual_tol=1e-10)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        iters = rec.converged_at if rec.converged_at is not None else (
            rec.diverged_at if rec.diverged else pb.max_iters)
        n_done = iters if iters else 1
        pts = phi_per_iteration(pb) * pb.n_x * n_done
        out.append(dict(case=pb.name, cfl=pb.cfl, m=pb.m, weno=pb.weno_order[0],
                        stepper=pb.stepper[0], relaxation=pb.relaxation,
                        iterations_to_tol=rec.converged_at, diverged_at=rec.diverged_at,
                        residuals=[None if r != r else r for r in rec.residuals.tolist()],
                        wall_s=wall, s_per_iter=wall / n_done,
                        point_updates_per_s=pts / wall))
        print(json.dumps(out[-1]), flush=True)
    print(json.dumps({"total_s": time.perf_counter() - t_all, "cases": len(out)}))


if __name__ == "__main__":
    main()

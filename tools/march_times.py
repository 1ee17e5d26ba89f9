"""Per-step time of single-field marches (us), WENO order x mesh x path:
Field path (MGP_MARCH2=0) and march_kernel at each cluster size."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09404_b200 as P  # noqa: E402
from paper_2104_09404_b200 import device as dev  # noqa: E402
from paper_2104_09404_b200._lib import G_NONE, SUM_LANE2  # noqa: E402

res = {}
n = 512
for order in (1, 3, 5):
    for nx in (64, 128, 256, 512, 1024, 2048, 4096):
        op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, nx),
                                    P.FluxConfig("lf", P.WenoConfig(order)))
        phi = P.RungeKuttaStepper(op.rhs, 0.2 / nx, 3).phi_struct(SUM_LANE2)
        x = (np.arange(nx) + 0.5) / nx
        traj = torch.empty(n + 1, nx, dtype=torch.float64, device="cuda")
        traj[0] = torch.from_numpy(0.5 + 0.25 * np.sin(2 * np.pi * x)).cuda()
        row = {}
        for name, env in [("field", {"MGP_MARCH2": "0"})] + \
                [(f"cs{c}", {"MGP_MARCH_CS": str(c)}) for c in (2, 4, 8, 16) if 8 <= nx // c <= 256]:
            os.environ.pop("MGP_MARCH2", None)
            os.environ.pop("MGP_MARCH_CS", None)
            os.environ.update(env)
            f = lambda: dev.sweep(phi, n_chunks=1, start=traj, start_stride=0, n_steps=n,
                                  g_mode=G_NONE, store=traj[1], st_ss=nx)
            f()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            row[name] = round(1e3 * a.elapsed_time(b) / n, 2)
        os.environ.pop("MGP_MARCH2", None)
        os.environ.pop("MGP_MARCH_CS", None)
        res[f"weno{order}_nx{nx}"] = row
        print(f"weno{order}_nx{nx}", json.dumps(row), flush=True)

"""Full-size MGRIT fixtures for BASELINE configs 4 and 5 (and the bench
relaxation), generated with the pinned CPU oracle -- TEST INFRASTRUCTURE.

Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py c4 c5
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_full.py refcheck

``c4``: every one of BASELINE config 4's 192 cases at full size (Burgers,
N_x = 1024, N_t = 16384, 3 levels, CFL x m x scheme x integrator x
relaxation), residual-only semantics, up to 10 iterations, stopping after the
first row below 1e-10 (the package driver's ``residual_tol``; the rows are a
prefix of the reference's ``mgrit_solve`` rows, mgrit.py:276-340).

``c5``: config-5-shaped runs at config 5's mesh (N_x = 65536, 16-mode a_k/k
IC, m = 16, WENO5 + SSP-RK3, FCF, V-cycles) with N_t reduced to 4096 and
L = 3 ("same Nx with Nt scaled down"): the CFL-0.4 case of
the config itself and a converging variant (CFL 0.4 / 256, coarsest CFL
0.4).

Per case the fixture keeps the residual rows, ``diverged_at``,
``converged_at`` and, after every recorded row, a SHA-256 of the whole
finest-level iterate (canonical bytes: every NaN as one bit pattern, -0.0 as
+0.0 -- the only representation differences DESIGN.md section 2 tolerates),
so the GPU tests check the trajectory bit for bit without storing it.

The oracle (``oracle/phi_oracle.c`` + ``oracle/mgrit_oracle.py``) is pinned
bit for bit against the unmodified reference by ``make_golden.py``; the
``refcheck`` mode re-runs a subset at full size through the unmodified
reference itself (``/root/reference/pkg/src``) and asserts the same rows
and iterates (``full_refcheck.json`` records what was checked).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from oracle import mgrit_oracle  # noqa: E402
from fixture_hash import canonical_hash  # noqa: E402
from paper_2104_09404_b200 import harness as H  # noqa: E402  (IC / grid helpers only)

_RK = {"fe": 1, "ssprk2": 2, "ssprk3": 3}
OUT_C4 = os.path.join(HERE, "full_c4.json")
OUT_C5 = os.path.join(HERE, "full_c5.json")
OUT_REF = os.path.join(HERE, "full_refcheck.json")


def c5_problems():
    base = H.BASELINE_CONFIGS["c5"].scaled(n_t=4096, n_levels=3, max_iters=2)
    return [base.scaled(name="c5-shaped-cfl0.4"),
            base.scaled(name="c5-shaped-cfl0.0015625", cfl=0.4 / 256, max_iters=3)]


def oracle_steppers(pb, tg, nthreads=0):
    orders = pb.weno_order * (pb.n_levels if len(pb.weno_order) == 1 else 1)
    kinds = pb.stepper * (pb.n_levels if len(pb.stepper) == 1 else 1)
    return [oracle.OracleStepper(k=(orders[l] - 1) // 2, rk_order=_RK[kinds[l]],
                                 dt=tg.dt * pb.m ** l, dx=pb.space_grid().dx,
                                 eps=pb.epsilon, nthreads=nthreads)
            for l in range(pb.n_levels)]


def run_oracle(pb, residual_tol):
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    st = oracle_steppers(pb, tg)
    hashes = []
    opts = mgrit_oracle.Options(n_levels=pb.n_levels, m=pb.m, cycle=pb.cycle,
                                relaxation=pb.relaxation, guess=pb.guess,
                                max_iters=pb.max_iters)
    hout = []
    t0 = time.perf_counter()
    _, rec = mgrit_oracle.mgrit_solve(
        st, u0, pb.n_t, tg.dt, opts, residual_tol=residual_tol, hierarchy_out=hout,
        on_row=lambda it, h: hashes.append(canonical_hash(h.fine_values())))
    final = canonical_hash(hout[0].fine_values())
    wall = time.perf_counter() - t0
    conv = None
    if residual_tol is not None:
        for it in range(1, len(rec.residuals)):
            if rec.residuals[it] < residual_tol:
                conv = it
                break
    return dict(name=pb.name, n_x=pb.n_x, n_t=pb.n_t, cfl=pb.cfl, m=pb.m,
                n_levels=pb.n_levels, weno=list(pb.weno_order), stepper=list(pb.stepper),
                relaxation=pb.relaxation, cycle=pb.cycle, guess=pb.guess,
                n_modes=pb.n_modes, decay=pb.decay, seed=pb.seed,
                max_iters=pb.max_iters, residual_tol=residual_tol,
                horizon=tg.horizon, dt=tg.dt,
                residuals=[None if not np.isfinite(r) else float(r) for r in rec.residuals],
                residual_repr=[repr(float(r)) for r in rec.residuals],
                diverged_at=rec.diverged_at, converged_at=conv,
                iterate_sha256=hashes, final_sha256=final, oracle_wall_s=wall)


def gen(out_path, problems, residual_tol):
    done = {}
    if os.path.exists(out_path):
        for c in json.load(open(out_path))["cases"]:
            done[c["name"]] = c
    for pb in problems:
        if pb.name in done:
            continue
        c = run_oracle(pb, residual_tol)
        done[pb.name] = c
        print(f"{pb.name}: conv={c['converged_at']} div={c['diverged_at']} "
              f"rows={c['residual_repr'][:3]} {c['oracle_wall_s']:.1f}s", flush=True)
        order = [p.name for p in problems if p.name in done]
        with open(out_path, "w") as f:
            json.dump({"generator": "tests/golden/make_golden_full.py (oracle C port)",
                       "cases": [done[n] for n in order]}, f, indent=0)


def refcheck(names):
    """Re-run cases through the unmodified reference (mgritlab) at full size
    and assert the oracle fixture's rows and iterate hashes."""
    sys.path.insert(0, "/root/reference/pkg/src")
    import mgritlab as R
    fixtures = {}
    for p in (OUT_C4, OUT_C5):
        if os.path.exists(p):
            for c in json.load(open(p))["cases"]:
                fixtures[c["name"]] = c
    problems = {pb.name: pb for pb in H.c4_grid() + c5_problems()}
    results = json.load(open(OUT_REF))["checked"] if os.path.exists(OUT_REF) else []
    seen = {r["name"] for r in results}
    for name in names:
        if name in seen:
            continue
        pb, fx = problems[name], fixtures[name]
        u0 = pb.initial_state()
        sg = R.SpatialGrid(pb.length, pb.n_x)
        tg = R.TemporalGrid(fx["horizon"], pb.n_t)
        assert tg.dt == fx["dt"]
        model = R.make_model("burgers")
        orders = pb.weno_order * (pb.n_levels if len(pb.weno_order) == 1 else 1)
        kinds = pb.stepper * (pb.n_levels if len(pb.stepper) == 1 else 1)
        steppers = [R.RungeKuttaStepper(
            R.SemiDiscreteOperator(model, sg, R.FluxConfig("lf", R.WenoConfig(
                order=orders[l], epsilon=pb.epsilon))).rhs, tg.dt * pb.m ** l, _RK[kinds[l]])
            for l in range(pb.n_levels)]
        # rows 0..n of the reference's own mgrit_solve, n = the fixture's last row
        n_rows = len([r for r in fx["residual_repr"] if r != "nan"])
        n_it = fx["diverged_at"] if fx["diverged_at"] is not None else n_rows - 1
        opts = R.MgritOptions(n_levels=pb.n_levels, m=pb.m, cycle=pb.cycle,
                              relaxation=pb.relaxation, guess=pb.guess, max_iters=n_it)
        t0 = time.perf_counter()
        traj, rec = R.mgrit_solve(steppers, u0, tg, sg, opts)
        wall = time.perf_counter() - t0
        got = [repr(float(r)) for r in rec.residuals]
        want = fx["residual_repr"][:len(got)]
        ok_rows = all(a == b or abs(float(a) - float(b)) <= 1e-12 * abs(float(b))
                      for a, b in zip(got, want) if b != "nan")
        assert ok_rows, (name, got, want)
        assert rec.diverged_at == fx["diverged_at"], (name, rec.diverged_at)
        h = canonical_hash(traj.values)
        assert h == fx["final_sha256"], name
        results.append(dict(name=name, rows=got, diverged_at=rec.diverged_at,
                            final_sha256=h,
                            reference_wall_s=wall))
        print(f"refcheck {name}: ok ({wall:.0f} s)", flush=True)
        with open(OUT_REF, "w") as f:
            json.dump({"generator": "tests/golden/make_golden_full.py refcheck "
                                    "(unmodified reference, /root/reference/pkg/src)",
                       "checked": results}, f, indent=1)


REFCHECK_DEFAULT = ["c4-cfl0.1-m2-weno1-ssprk3-fcf", "c4-cfl0.2-m2-weno3-ssprk2-f",
                    "c4-cfl0.4-m4-weno5-ssprk3-fcf", "c4-cfl0.8-m16-weno3-ssprk3-f"]


if __name__ == "__main__":
    which = sys.argv[1:] or ["c4", "c5"]
    if "c4" in which:
        gen(OUT_C4, [pb.scaled(max_iters=10) for pb in H.c4_grid()], 1e-10)
    if "c5" in which:
        gen(OUT_C5, c5_problems(), None)
    if "refcheck" in which:
        rest = [w for w in which if w not in ("c4", "c5", "refcheck")]
        refcheck(rest or REFCHECK_DEFAULT)

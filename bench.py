#!/usr/bin/env python
"""Benchmark of the MGRIT fine-propagator path (BASELINE.json metric:
fine space-time point-updates/s of the WENO5 + SSP-RK3 propagator in MGRIT
relaxation; s/iter).

Workload (default, BASELINE.json configs[2], "c3" -- the largest
single-GPU configuration): 1D Burgers, N_x = 4096, N_t = 65536, CFL 0.4,
WENO5-JS (eps 1e-6) + global LF + SSP-RK3, fp64, seeded 8-mode Fourier IC
(seed 1234), m = 4, 7 levels, FCF relaxation.  One step = one complete FCF
relaxation of the finest level over all 16384 CF-intervals, F-points
written to HBM: (2m - 1) * N_t/m * N_x = 469,762,048 point-updates, exactly
the propagator applications of the reference's relax(0) (mgrit.py:193-197).
The input iterate is the serial solution's C-points (finite data); each step
relaxes the previous step's output.  The 126 MB L2 is flushed between steps
(outside the timed region; the step's own input, 537 MB of C-points, is
larger than L2 anyway).  ``iteration_ms`` times one whole V-cycle iteration
+ residual row of the same config from its initial iterate (the reference's
MGRIT iteration 1, mgrit.py:315-332).  ``--workload c2`` keeps round 1's
configs[1] line.

``--impl reference`` times the CPU oracle port (oracle/, a bit-exact C
restatement of the reference propagator and MGRIT driver, all host threads):
each step is a bounded sample -- the FCF relaxation of the first 1024
CF-intervals of the same finest level (29.4 M point-updates) -- and
``iteration_ms`` is one whole V-cycle + residual row of the full config,
timed once.  The reference itself is Python/NumPy and is not installable on
the GPU box.
"""
from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse  # noqa: E402
import ctypes  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "point-updates/s"
FLOPS_PER_PT = {  # literal FP64 add/sub/mul/div per point-update
    (2, 3): 735, (2, 2): 489, (1, 3): 297, (1, 2): 197, (0, 3): 45, (0, 2): 29, (0, 1): 13}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c2", "c3", "c4"])
    ap.add_argument("--no-cpu-iteration", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def workload(name):
    import paper_2104_09404_b200 as P
    pb = P.BASELINE_CONFIGS[name]
    if name == "c4":  # heaviest C4 case: WENO5 / SSP-RK3, m = 2, FCF
        pb = pb.scaled(m=2, weno_order=(5,), stepper=("ssprk3",), relaxation="fcf")
    return pb


def relax_units(pb) -> int:
    return (2 * pb.m - 1) * (pb.n_t // pb.m) * pb.n_x


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU arm (oracle port)
# ---------------------------------------------------------------------------

CPU_SAMPLE_INTERVALS = 1024


def cpu_relax_setup(pb):
    """The oracle port on a bounded sample of the workload: a 2-level
    hierarchy over the first CPU_SAMPLE_INTERVALS CF-intervals of the
    finest level, holding the serial trajectory there (finite data, as the
    GPU arm); its relax(0) is the reference's FCF relaxation of those
    intervals (mgrit.py:193-197)."""
    import oracle
    from oracle import mgrit_oracle
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    p = pb.phi_params(0)
    nthreads = oracle.lib().ora_max_threads()
    st = oracle.OracleStepper(model=p["model"], k=p["k"], rk_order=p["rk_order"],
                              dt=p["dt"], dx=p["dx"], eps=p["eps"], speed=p["speed"],
                              nthreads=nthreads)
    nci = min(CPU_SAMPLE_INTERVALS, pb.n_t // pb.m)
    h = mgrit_oracle.Hierarchy([st, st], u0, nci * pb.m, tg.dt,
                               mgrit_oracle.Options(n_levels=2, m=pb.m, relaxation="fcf"))
    h.levels[0].u[:] = mgrit_oracle.march(st, u0, nci * pb.m)
    return h, nthreads, (2 * pb.m - 1) * nci * pb.n_x, nci


def cpu_relax_rate(pb, seconds: float):
    h, nthreads, units, _ = cpu_relax_setup(pb)
    done, t0 = 0, time.perf_counter()
    while True:
        h.relax(0)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return units * done / el, nthreads, done, el


def cpu_iteration_ms(pb):
    """One whole MGRIT iteration of the full config on the oracle port
    (run_cycle + residual_norm from the initial iterate, mgrit.py:315-322),
    the CPU side of ``iteration_ms``."""
    import oracle
    from oracle import mgrit_oracle
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    nthreads = oracle.lib().ora_max_threads()
    st = []
    for l in range(pb.n_levels):
        p = pb.phi_params(l)
        st.append(oracle.OracleStepper(model=p["model"], k=p["k"], rk_order=p["rk_order"],
                                       dt=p["dt"], dx=p["dx"], eps=p["eps"],
                                       speed=p["speed"], nthreads=nthreads))
    h = mgrit_oracle.Hierarchy(st, u0, pb.n_t, tg.dt,
                               mgrit_oracle.Options(n_levels=pb.n_levels, m=pb.m,
                                                    relaxation=pb.relaxation))
    with np.errstate(all="ignore"):
        t0 = time.perf_counter()
        h.run_cycle()
        r = h.residual_norm()
        el = time.perf_counter() - t0
    return 1e3 * el, r, nthreads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pb = workload(args.workload)
    h, nthreads, units, nci = cpu_relax_setup(pb)
    for _ in range(args.warmup):
        h.relax(0)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        h.relax(0)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = units * args.steps / total
    sample = (f"per step: FCF relaxation of the first {nci} of {pb.n_t // pb.m} "
              f"CF-intervals of the finest level ({units} point-updates), "
              f"oracle C port, {nthreads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(pb, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_iteration:
        it_ms, r, _ = cpu_iteration_ms(pb)
        line["iteration_ms"] = it_ms
        line["iteration_note"] = (f"one whole V-cycle ({pb.n_levels} levels, FCF) + residual "
                                  f"row of the full config from the initial iterate, oracle "
                                  f"port, {nthreads} threads (residual after: {r})")
    print(json.dumps(line), flush=True)


def config_block(pb, args):
    return {"workload": f"{args.workload}: {pb.name}", "n_x": pb.n_x, "n_t": pb.n_t,
            "m": pb.m, "n_levels": pb.n_levels, "relaxation": "fcf",
            "scheme": f"WENO{pb.weno_order[0]}+{pb.stepper[0]}+global-LF",
            "cfl": pb.cfl, "seed": pb.seed,
            "step": "one FCF relaxation of the finest level, all CF-intervals, "
                    "F-points stored",
            "point_updates_per_step": relax_units(pb),
            "l2": "flushed (256 MiB write) between timed steps",
            "input": "serial solution's C-points (finite data), resident in HBM"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def fp64_peak():
    path = os.path.join(ROOT, "tools", "libfp64probe.so")
    if not os.path.exists(path):
        return None, None
    lib = ctypes.CDLL(path)
    lib.fp64_probe.restype = ctypes.c_double
    lib.fp64_probe.argtypes = [ctypes.c_int, ctypes.c_int]
    addmul = lib.fp64_probe(0, 4000)
    fma = lib.fp64_probe(1, 4000)
    return (addmul if addmul > 0 else None), (fma if fma > 0 else None)


def load_profile_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2104_09404_b200 as P
    from paper_2104_09404_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pb = workload(args.workload)
    u0 = pb.initial_state()
    tg1 = pb.time_grid(u0)
    sg = pb.space_grid()
    units = relax_units(pb)              # per rank (weak scaling: fixed per-GPU work)
    k = (pb.weno_order[0] - 1) // 2
    rk = {"fe": 1, "ssprk2": 2, "ssprk3": 3}[pb.stepper[0]]
    flops_pt = FLOPS_PER_PT.get((k, rk))
    nc = pb.n_t // pb.m

    # finite input iterate: the serial solution's C-points (this rank's slab)
    steppers1 = pb.steppers(tg1)
    serial = P.serial.march(steppers1[0], u0, pb.n_t)
    force_dist = os.environ.get("MGP_FORCE_DIST") == "1"   # exercise the N>1 path on 1 GPU
    if world == 1 and force_dist and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    if world == 1 and not force_dist:
        tg, steppers = tg1, steppers1
        h = P.MgritHierarchy(steppers, u0, tg, sg, pb.options())
    else:
        # weak scaling: the time axis grows with the number of GPUs, each rank
        # owning the same 1024 CF-intervals; one boundary state is exchanged
        # per C-relaxation (distributed.py)
        from paper_2104_09404_b200.distributed import DistMgritHierarchy
        tg = P.TemporalGrid(tg1.horizon * world, pb.n_t * world)
        steppers = P.build_steppers(pb.model_obj(), sg, tg, n_levels=pb.n_levels, m=pb.m,
                                    weno_order=pb.weno_order, stepper=pb.stepper,
                                    epsilon=pb.epsilon)
        h = DistMgritHierarchy(steppers, u0, tg, sg, pb.options())
    h.load_c_points(serial[::pb.m, 0])
    traj = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    dist_path = world > 1 or force_dist

    def materialise(out):
        if not dist_path:
            return h.fine_values(out=out)
        out.view(-1, pb.n_x).copy_(h._local_values())
        return out

    # N = 1 and N > 1 run the same fused kernel (distributed.py
    # relax_fine_values: the local intervals, then the boundary exchange)
    fused = h._fcf_workspace() is not None
    h._fcf_segment = int(os.environ.get("MGP_BENCH_SEGMENT", "0"))   # tuning experiments
    h._fcf_split = int(os.environ.get("MGP_BENCH_SPLIT", "0"))       # 0 = automatic plan

    def step(record_kernels=False):
        if fused:
            # ONE launch: every interval's F- and C-steps, then the next
            # interval's final F-steps with the F-points stored, split over
            # persistent CTAs by step (mgp_relax_fcf)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
            h.relax_fine_values(out=traj)
            e[1].record(stream)
            e[2], e[3] = e[0], e[0]
            return e
        if record_kernels:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
            h.c_relax(0)          # fused F + C (m steps per chunk)
            e[1].record(stream)
            h.f_relax(0)
            e[2].record(stream)
            materialise(traj)     # F-relax with every F-point stored
            e[3].record(stream)
            return e
        h.relax(0)
        materialise(traj)
        return None

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    launches0 = _lib.launch_count()
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    kevents = []
    for _ in range(args.steps):
        flush.zero_()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        ev = step(record_kernels=True)
        s1.record(stream)
        kevents.append(ev)
        step_ms.append((s0, s1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop() if clocks else None
    launches = _lib.launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in step_ms)
    step_total_ms = total_ms
    k_fc = [ev[0].elapsed_time(ev[1]) for ev in kevents]
    k_f = [ev[2].elapsed_time(ev[3]) for ev in kevents]
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = units * args.steps * world / (total_ms * 1e-3)

    # ---- end to end through the public API with host buffers --------------
    # relax_to_host: C-points host->device, FCF relaxation, trajectory
    # device->host, the copies pipelined against the kernels (mgrit.py)
    # pieces of the pipelined relax_to_host: default = the API's own choice
    # (zero-copy launch for small configs, 64 pipelined pieces at config 3)
    e2e_pieces = int(os.environ["MGP_E2E_PIECES"]) if "MGP_E2E_PIECES" in os.environ else None
    e2e_graph = os.environ.get("MGP_E2E_GRAPH", "0") == "1"
    host_in = torch.empty(nc + 1, pb.n_x, dtype=torch.float64).pin_memory()
    host_in.copy_(serial[::pb.m, 0].cpu())
    host_out = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if not dist_path:
            h.relax_to_host(host_in, host_out, pieces=e2e_pieces, graph=e2e_graph)
        else:
            # the rank's fused launch on its mapped pinned buffers + the
            # boundary exchange (DistMgritHierarchy.relax_to_host)
            h.relax_to_host(host_in, host_out)
        b.record(stream)
        if i >= args.warmup:
            e2e_ms.append((a, b))
    torch.cuda.synchronize()
    e2e_total = sum(a.elapsed_time(b) for a, b in e2e_ms)
    # the pipelined step must equal the unpipelined public-API result
    h.load_c_points(host_in)
    h.relax(0)
    if not dist_path:
        assert torch.equal(materialise(traj).cpu(), host_out), "relax_to_host mismatch"
    te = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units * args.steps * world / (float(te.item()) * 1e-3)

    # ---- one whole MGRIT iteration (V-cycle + residual) from the IC --------
    it_ms = []
    for i in range(4):
        if not dist_path:
            hi = P.MgritHierarchy(steppers, u0, tg, sg, pb.options())
        else:
            from paper_2104_09404_b200.distributed import DistMgritHierarchy
            hi = DistMgritHierarchy(steppers, u0, tg, sg, pb.options())
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        hi.run_cycle()
        mon = hi.monitor()
        b.record(stream)
        torch.cuda.synchronize()
        if i:
            it_ms.append(a.elapsed_time(b))

    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    peak_addmul, peak_fma = fp64_peak()
    prof = load_profile_traffic()
    kernel_ms = sum(k_fc) + sum(k_f)
    kernel_units = (pb.m * nc * pb.n_x + (pb.m - 1) * nc * pb.n_x) * args.steps
    achieved = flops_pt * kernel_units / (kernel_ms * 1e-3) / 1e12 if flops_pt else None
    row_b = 8 * pb.n_x
    if fused:
        kname = f"fcf_kernel<{k},burgers> (fused FCF relaxation, F-points stored)"
        # C-points read, new C-points written twice (C-point buffer and
        # trajectory rows), F-points written
        alg_bytes = {"fcf": row_b * ((nc + 1) + nc + (nc + 1) + nc * (pb.m - 1))}
    else:
        kname = f"sweep_kernel<{k},burgers> (fused F/C relaxation)"
        alg_bytes = {"fused_f_c": 16 * nc * pb.n_x, "f_store": 8 * pb.m * nc * pb.n_x}
    roofline = {
        "bound": "fp64",
        "kernel": kname,
        "achieved": achieved, "unit": "TFLOP/s",
        "peak": peak_addmul / 1e12 if peak_addmul else None,
        "peak_source": "measured: tools/fp64_peak.cu DADD/DMUL issue rate, 1 op = 1 flop "
                       "(MEASURED_PEAKS.json has no FP64 figure)",
        "frac": (achieved / (peak_addmul / 1e12)) if (achieved and peak_addmul) else None,
        "peak_fma": 2 * peak_fma / 1e12 if peak_fma else None,
        "frac_of_fma_peak": (achieved / (2 * peak_fma / 1e12)) if (achieved and peak_fma) else None,
        "flops_per_point_update": flops_pt,
        "kernel_share_of_step": kernel_ms / step_total_ms if step_total_ms else None,
        "traffic": prof.get("dram_bytes_per_launch"),
        "algorithmic_bytes_per_launch": alg_bytes,
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(pb, args),
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": host_in.numel() * 8,
                "d2h_bytes_per_step": host_out.numel() * 8},
        "gpu_launches": launches,
        "clocks": clock_info,
        "iteration_ms": statistics.median(it_ms),
        "iteration_note": f"one V-cycle (FCF, {pb.n_levels} levels, "
                          f"{pb.n_t // pb.m ** (pb.n_levels - 1)}-step sequential coarse solve) "
                          "+ residual row from the initial iterate, median of 3 "
                          f"(residual after: {mon.residual})",
        "kernel_ms": ({"fcf": statistics.median(k_fc)} if fused else
                      {"fused_f_c": statistics.median(k_fc), "f_store": statistics.median(k_f)}),
    }
    if world == 1 and not force_dist and args.workload != "c2":
        line["config2"] = side_workload("c2", flush, stream)   # round 1's bench workload, for context
    if not args.no_cpu_baseline and world == 1:
        rate, cores, n, el = cpu_relax_rate(pb, args.cpu_seconds)
        nci = min(CPU_SAMPLE_INTERVALS, nc)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{n} FCF relaxation(s) of the first {nci} of {nc} "
                                          f"CF-intervals of the same finest level in "
                                          f"{el:.1f} s (oracle C port)"}
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def side_workload(name, flush, stream, steps=20):
    """The same step and iteration on another BASELINE config (device-timed
    only), reported as extra keys next to the headline workload."""
    import torch

    import paper_2104_09404_b200 as P
    pb = workload(name)
    u0 = pb.initial_state()
    tg = pb.time_grid(u0)
    sg = pb.space_grid()
    steppers = pb.steppers(tg)
    serial = P.serial.march(steppers[0], u0, pb.n_t)
    h = P.MgritHierarchy(steppers, u0, tg, sg, pb.options())
    h.load_c_points(serial[::pb.m, 0])
    traj = torch.empty(pb.n_t + 1, 1, pb.n_x, dtype=torch.float64, device="cuda")
    for _ in range(3):
        h.relax_fine_values(out=traj)
    ev = []
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        h.relax_fine_values(out=traj)
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    it = []
    for i in range(4):
        hi = P.MgritHierarchy(steppers, u0, tg, sg, pb.options())
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        hi.run_cycle()
        hi.monitor()
        b.record(stream)
        torch.cuda.synchronize()
        if i:
            it.append(a.elapsed_time(b))
    return {"workload": f"{name}: {pb.name}", "value": relax_units(pb) / (ms * 1e-3),
            "unit": UNIT, "ms_per_step": ms, "iteration_ms": statistics.median(it),
            "point_updates_per_step": relax_units(pb)}


def main():
    args = parse()
    # stdout carries exactly one JSON line: anything a library prints on file
    # descriptor 1 meanwhile (NCCL's version banner) goes to stderr instead
    sys.stdout.flush()
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(real_stdout, "w", buffering=1)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    sys.stdout.flush()


if __name__ == "__main__":
    main()

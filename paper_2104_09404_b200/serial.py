"""Sequential time marching on the GPU: the reference trajectory each
parallel solve is held to (reference ``pkg/src/mgritlab/serial.py``).

``solve_serial`` marches the single state through every node with one
persistent CTA (``mgp_sweep`` with one chunk, every step stored), in the
single-field summation regime the reference's ``advance((D, N))`` calls use.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import device as dev
from ._lib import G_NONE
from .errors import DimensionError
from .grid import SpatialGrid, TemporalGrid, Trajectory


@dataclass
class SerialRun:
    """serial.py:15-21; trajectory.values is a host array, ``device_values``
    the same trajectory on the GPU."""

    trajectory: Trajectory
    max_speed: float
    max_cfl: float
    wall_seconds: float
    device_values: object = None


def discretise_ic(ic, space_grid: SpatialGrid) -> np.ndarray:
    """Sample a pointwise initial condition at cell midpoints (serial.py:24-37)."""
    values = np.asarray(ic(space_grid.cell_centers()), float)
    if values.ndim == 1:
        values = values[None, :]
    if values.ndim != 2 or values.shape[1] != space_grid.n_cells:
        raise DimensionError(f"initial condition produced shape {values.shape} on a "
                             f"{space_grid.n_cells}-cell mesh")
    return values


def march(stepper, initial_state, n_steps: int) -> torch.Tensor:
    """Device trajectory (n_steps + 1, D, N): u[i] = Phi(u[i-1])."""
    D = getattr(stepper, "n_components", 1)
    u0 = dev.to_device(initial_state).reshape(-1)
    nx = u0.numel()
    if nx != D * stepper.nx:
        raise DimensionError(f"initial state has {nx} values, the stepper works on "
                             f"({D}, {stepper.nx}) states")
    out = torch.empty(n_steps + 1, nx, dtype=dev.DTYPE, device=u0.device)
    out[0].copy_(u0)
    if n_steps:
        dev.sweep(stepper.phi_struct(dev.regime_for_batch(1)), n_chunks=1,
                  start=out, start_stride=0, n_steps=n_steps, g_mode=G_NONE,
                  store=out[1], st_ss=nx, what="solve_serial")
        if D > 1:
            dev.check_status()
    return out.view(n_steps + 1, D, nx // D)


def solve_serial(stepper, initial_state, time_grid: TemporalGrid,
                 space_grid: SpatialGrid, model=None) -> SerialRun:
    """March the initial state across every node of the time grid
    (serial.py:40-61)."""
    start = time.perf_counter()
    values = march(stepper, initial_state, time_grid.n_steps)
    max_speed = 0.0
    if model is not None:
        if getattr(model, "kind", "") == "advection":
            max_speed = abs(model.speed)
        elif getattr(model, "kind", "") in ("shallow-water", "euler"):
            # serial.py:47-54: running max over nodes of max |u| + sqrt(g h)
            # (Python max ignores NaN nodes after the first)
            if model.kind == "shallow-water":
                h, hu = values[:, 0, :], values[:, 1, :]
                speed = (hu / h).abs() + torch.sqrt(model.gravity * h)
            else:
                rho, mom, en = values[:, 0, :], values[:, 1, :], values[:, 2, :]
                vel = mom / rho
                p = (model.gamma - 1.0) * (en - ((0.5 * rho) * vel) * vel)
                speed = vel.abs() + torch.sqrt((model.gamma * p) / rho)
            per_node = speed.amax(dim=1)
            per_node = torch.where(torch.isnan(per_node), torch.zeros_like(per_node),
                                   per_node)
            max_speed = float(per_node.max().item())
        else:
            per_node = values.abs().amax(dim=(1, 2))
            per_node = torch.where(torch.isnan(per_node), torch.zeros_like(per_node),
                                   per_node)
            max_speed = float(per_node.max().item())
    if values.is_cuda:
        torch.cuda.synchronize()
    wall = time.perf_counter() - start
    trajectory = Trajectory(time_grid, space_grid, values.cpu().numpy())
    cfl = max_speed * time_grid.dt / space_grid.dx
    return SerialRun(trajectory=trajectory, max_speed=max_speed, max_cfl=cfl,
                     wall_seconds=wall, device_values=values)

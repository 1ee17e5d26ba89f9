"""Propagators on the GPU.

Mirrors reference ``pkg/src/mgritlab/stepper.py``:

* ``RungeKuttaStepper(rhs, dt, order)`` (stepper.py:68-82); ``rhs`` must be the
  bound ``rhs`` of this package's :class:`SemiDiscreteOperator`, whose
  parameters the fused kernel consumes (the stages run inside one kernel).
* the one-step Lax-Friedrichs family of the paper's coarse operators,
  Burgers only: ``MatchedLFFine`` (:102-114), ``MatchedLFCoarse`` order 0/1
  (:117-152), ``RediscretizedLF`` (:155-167);
* ``ComposedStepper(inner, repeats)`` (:170-188), the exact m-fold
  composition, for any of the above;
* ``StepperSpec`` / ``make_stepper`` (:191-231), ``neighbor_average`` /
  ``central_difference`` (:85-92, host NumPy helpers).

Every ``advance(u)`` runs on the GPU (one ``mgp_sweep`` launch); NumPy in ->
NumPy out, CUDA tensor in -> tensor out.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import MgpPhi, SCHEME_LF_MATCHED, SCHEME_LF_ONESTEP
from .errors import ConfigError
from .flux import SemiDiscreteOperator, apply_phi, apply_phi_struct
from .models import Burgers

STEPPER_KINDS = ("fe", "ssprk2", "ssprk3", "matched-lf-fine", "matched-lf-0",
                 "matched-lf-1", "rediscretized-lf")
_RK_ORDERS = {"fe": 1, "ssprk2": 2, "ssprk3": 3}


class RungeKuttaStepper:
    """SSP Runge-Kutta time stepper around a semi-discrete operator."""

    def __init__(self, rhs, dt: float, order: int):
        if order not in (1, 2, 3):
            raise ConfigError(f"no Runge-Kutta stepper of order {order}")
        if dt <= 0.0:
            raise ConfigError(f"time step must be positive, got {dt}")
        op = getattr(rhs, "__self__", None)
        if not isinstance(op, SemiDiscreteOperator) or rhs.__func__ is not SemiDiscreteOperator.rhs:
            raise ConfigError("the B200 RungeKuttaStepper needs the rhs of a "
                              "paper_2104_09404_b200.SemiDiscreteOperator")
        self.rhs = rhs
        self.operator = op
        self.dt = dt
        self.order = order

    def advance(self, u):
        """One step on every (D, N) field of u (stepper.py:81-82).  NumPy in
        -> NumPy out; CUDA tensor in -> CUDA tensor out."""
        return apply_phi(self.operator, self.dt, self.order, u)

    def phi_struct(self, regime: int):
        return self.operator.phi_struct(dt=self.dt, rk_order=self.order, regime=regime)

    @property
    def nx(self) -> int:
        return self.operator.space_grid.n_cells

    @property
    def n_components(self) -> int:
        return self.operator.n_components


def neighbor_average(u):
    """E(u)_i = (u_{i+1} + u_{i-1}) / 2 on the periodic last axis (host)."""
    return 0.5 * (np.roll(u, -1, axis=-1) + np.roll(u, 1, axis=-1))


def central_difference(f, dx: float):
    """D(f)_i = (f_{i+1} - f_{i-1}) / (2 dx) on the periodic last axis (host)."""
    return (np.roll(f, -1, axis=-1) - np.roll(f, 1, axis=-1)) / (2.0 * dx)


def _require_scalar_model(model, kind: str) -> None:
    if not isinstance(model, Burgers):
        raise ConfigError(f"stepper '{kind}' is defined for the scalar model only, "
                          f"got '{getattr(model, 'kind', model)}'")


class _LFStepper:
    """Shared GPU plumbing of the one-step LF family."""

    scheme = SCHEME_LF_ONESTEP
    lf_order = 0
    m_effective = 1
    n_components = 1

    def _formula_dt(self) -> float:
        return self.dt

    def phi_struct(self, regime: int) -> MgpPhi:
        return MgpPhi(int(self.model.abi_model), 0, 1, int(regime), int(self.nx),
                      float(self._formula_dt()), float(self.dx), 1e-6, 0.0,
                      int(self.scheme), int(self.lf_order), int(self.m_effective), 1)

    def advance(self, u):
        return apply_phi_struct(self.phi_struct, self.nx, u)


class MatchedLFFine(_LFStepper):
    """One-step Lax-Friedrichs scheme Phi(u) = E u - dt D f(u) (stepper.py:102-114)."""

    def __init__(self, model, space_grid, dt: float):
        _require_scalar_model(model, "matched-lf-fine")
        self.model = model
        self.dx = space_grid.dx
        self.nx = space_grid.n_cells
        self.dt = dt


class RediscretizedLF(MatchedLFFine):
    """The fine one-step scheme rebuilt with the coarse step (stepper.py:155-167)."""

    def __init__(self, model, space_grid, dt: float):
        _require_scalar_model(model, "rediscretized-lf")
        super().__init__(model, space_grid, dt)


class MatchedLFCoarse(_LFStepper):
    """Truncated expansion of Phi^m (stepper.py:117-152)."""

    scheme = SCHEME_LF_MATCHED

    def __init__(self, model, space_grid, dt_fine: float, m_effective: int, order: int):
        _require_scalar_model(model, f"matched-lf-{order}")
        if order not in (0, 1):
            raise ConfigError(f"matched coarse operators exist for orders 0 and 1, got {order}")
        if m_effective < 1:
            raise ConfigError(f"m_effective must be >= 1, got {m_effective}")
        self.model = model
        self.dx = space_grid.dx
        self.nx = space_grid.n_cells
        self.dt_fine = dt_fine
        self.m_effective = m_effective
        self.order = order
        self.lf_order = order
        self.dt = dt_fine * m_effective

    def _formula_dt(self) -> float:
        # order 0 multiplies D f(u) by self.dt, order 1 the sum by dt_fine
        return self.dt if self.order == 0 else self.dt_fine


class ComposedStepper:
    """Exact repeats-fold composition of another stepper (stepper.py:170-188)."""

    def __init__(self, inner, repeats: int):
        if repeats < 1:
            raise ConfigError(f"repeats must be >= 1, got {repeats}")
        if not hasattr(inner, "phi_struct"):
            raise ConfigError("ComposedStepper needs a propagator of this package")
        self.inner = inner
        self.repeats = repeats
        self.dt = inner.dt * repeats
        self.nx = inner.nx
        self.n_components = getattr(inner, "n_components", 1)

    @property
    def operator(self):
        return getattr(self.inner, "operator", None)

    def phi_struct(self, regime: int) -> MgpPhi:
        p = self.inner.phi_struct(regime)
        p.repeats = int(p.repeats) * int(self.repeats)
        return p

    def advance(self, u):
        return apply_phi_struct(self.phi_struct, self.nx, u, self.n_components)


@dataclass(frozen=True)
class StepperSpec:
    """Names a stepper kind (stepper.py:191-211)."""

    kind: str
    m_effective: int = 1

    def __post_init__(self):
        if self.kind not in STEPPER_KINDS:
            raise ConfigError(f"unknown stepper kind '{self.kind}', "
                              f"expected one of {STEPPER_KINDS}")

    @property
    def order(self) -> int:
        if self.kind in _RK_ORDERS:
            return _RK_ORDERS[self.kind]
        if self.kind == "matched-lf-0":
            return 0
        return 1


def make_stepper(spec: StepperSpec, model, space_grid, dt: float, rhs=None):
    """Build the stepper named by spec (stepper.py:214-231)."""
    if spec.kind in _RK_ORDERS:
        if rhs is None:
            raise ConfigError(f"stepper '{spec.kind}' needs a right-hand side")
        return RungeKuttaStepper(rhs, dt, _RK_ORDERS[spec.kind])
    if spec.kind == "matched-lf-fine":
        return MatchedLFFine(model, space_grid, dt)
    if spec.kind == "rediscretized-lf":
        return RediscretizedLF(model, space_grid, dt)
    order = 0 if spec.kind == "matched-lf-0" else 1
    return MatchedLFCoarse(model, space_grid, dt, spec.m_effective, order)

"""SSP Runge-Kutta propagators on the GPU.

Mirrors reference ``pkg/src/mgritlab/stepper.py:68-82``: ``RungeKuttaStepper(
rhs, dt, order)`` with ``advance(u)``; ``rhs`` must be the bound ``rhs`` of
this package's :class:`SemiDiscreteOperator`, whose parameters the fused
kernel consumes (the stages run inside one kernel, never as separate rhs
calls).  Matched / rediscretised / composed LF steppers (stepper.py:85-188)
are the "next" row of SURVEY.md 8(f) and are rejected for now.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError
from .flux import SemiDiscreteOperator, apply_phi

STEPPER_KINDS = ("fe", "ssprk2", "ssprk3")
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
        """One step on every (1, N) field of u (stepper.py:81-82).  NumPy in
        -> NumPy out; CUDA tensor in -> CUDA tensor out."""
        return apply_phi(self.operator, self.dt, self.order, u)

    def phi_struct(self, regime: int):
        return self.operator.phi_struct(dt=self.dt, rk_order=self.order, regime=regime)

    @property
    def nx(self) -> int:
        return self.operator.space_grid.n_cells


@dataclass(frozen=True)
class StepperSpec:
    kind: str
    m_effective: int = 1

    def __post_init__(self):
        if self.kind not in STEPPER_KINDS:
            raise ConfigError(f"stepper kind '{self.kind}' is not on the B200 path; "
                              f"expected one of {STEPPER_KINDS}")

    @property
    def order(self) -> int:
        return _RK_ORDERS[self.kind]


def make_stepper(spec: StepperSpec, model, space_grid, dt: float, rhs=None):
    """stepper.py:214-231 for the Runge-Kutta kinds."""
    if rhs is None:
        raise ConfigError(f"stepper '{spec.kind}' needs a right-hand side")
    return RungeKuttaStepper(rhs, dt, _RK_ORDERS[spec.kind])

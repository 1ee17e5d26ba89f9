"""Scalar conservation-law models of the GPU path.

``Burgers`` mirrors reference ``pkg/src/mgritlab/models.py:101-133`` (flux
(0.5 u) u, eigenvalue u, max speed |u|).  ``Advection`` is the linear model
BASELINE.json config 1 needs (u_t + a u_x = 0, flux a u, |lambda| = |a|);
the reference rejects "advection" (tests/test_models.py:197-198), so it is a
new ``ConservationModel`` subclass with the same shape contract.
``ShallowWater`` (models.py:136-211, state (h, hu), gravity g) and ``Euler``
(models.py:214-308, state (rho, rho u, E), ratio gamma) run on the
characteristic-WENO system kernel.  Euler's left eigenvectors are the
inverse of the right ones; the reference takes it with LAPACK
(``np.linalg.inv``), the kernel with LU + partial pivoting in LAPACK's
operation order, so Euler results agree with the reference to rounding
(DESIGN.md "Euler parity"), shallow water bit for bit.

These host methods are the reference's NumPy semantics for callers and
tests; the device kernels implement the same formulas (csrc/mgrit_phi.cu).
"""
from __future__ import annotations

import numpy as np

from .errors import ConfigError, DimensionError, PhysicalStateError

MODEL_BURGERS = 0         # MGP_MODEL_BURGERS
MODEL_ADVECTION = 1       # MGP_MODEL_ADVECTION
MODEL_SHALLOW_WATER = 2   # MGP_MODEL_SHALLOW_WATER
MODEL_EULER = 3           # MGP_MODEL_EULER
DEFAULT_GRAVITY = 9.81    # models.py:21
DEFAULT_GAMMA = 5.0 / 3.0  # models.py:22


class ConservationModel:
    """Common interface (models.py:61-98)."""

    kind: str
    n_components: int
    abi_model: int

    def _check_shape(self, u) -> None:
        if u.ndim < 2 or u.shape[-2] != self.n_components:
            raise DimensionError(
                f"{self.kind} expects (..., {self.n_components}, N) states, "
                f"got shape {u.shape}")

    def flux(self, u):
        raise NotImplementedError

    def eigenvalues(self, u):
        raise NotImplementedError

    def max_abs_speed(self, u):
        return np.max(np.abs(self.eigenvalues(u)), axis=-1)


class Burgers(ConservationModel):
    """Scalar model with flux u^2/2; the single wave moves at speed u."""

    kind = "burgers"
    n_components = 1
    abi_model = MODEL_BURGERS
    speed = 0.0

    def flux(self, u):
        self._check_shape(u)
        return 0.5 * u * u

    def eigenvalues(self, u):
        self._check_shape(u)
        return np.moveaxis(u, -2, -1)

    def max_abs_speed(self, u):
        self._check_shape(u)
        return np.abs(u[..., 0, :])


class Advection(ConservationModel):
    """Linear advection u_t + a u_x = 0 with constant speed a."""

    kind = "advection"
    n_components = 1
    abi_model = MODEL_ADVECTION

    def __init__(self, speed: float = 1.0):
        speed = float(speed)
        if not np.isfinite(speed):
            raise ConfigError(f"advection speed must be finite, got {speed}")
        self.speed = speed

    def flux(self, u):
        self._check_shape(u)
        return self.speed * u

    def eigenvalues(self, u):
        self._check_shape(u)
        return np.full(np.moveaxis(u, -2, -1).shape, self.speed)

    def max_abs_speed(self, u):
        self._check_shape(u)
        return np.full(u[..., 0, :].shape, abs(self.speed))


class ShallowWater(ConservationModel):
    """Depth/momentum system (h, hu) with gravity wave speeds u -+ sqrt(g h)
    (models.py:136-183)."""

    kind = "shallow-water"
    n_components = 2
    abi_model = MODEL_SHALLOW_WATER
    speed = 0.0

    def __init__(self, gravity: float = DEFAULT_GRAVITY):
        if not gravity > 0.0:
            raise PhysicalStateError(f"gravity must be positive, got {gravity}")
        self.gravity = float(gravity)

    def _depth_velocity(self, u):
        h = u[..., 0, :]
        bad = h <= 0.0
        if np.any(bad):
            raise PhysicalStateError(
                f"non-positive depth in cell {int(np.argmax(bad.reshape(-1)))}")
        return h, u[..., 1, :] / h

    def flux(self, u):
        self._check_shape(u)
        h, vel = self._depth_velocity(u)
        return np.stack([u[..., 1, :], h * vel * vel + 0.5 * self.gravity * h * h],
                        axis=-2)

    def eigenvalues(self, u):
        self._check_shape(u)
        h, vel = self._depth_velocity(u)
        c = np.sqrt(self.gravity * h)
        return np.stack([vel - c, vel + c], axis=-1)

    def max_abs_speed(self, u):
        self._check_shape(u)
        h, vel = self._depth_velocity(u)
        return np.abs(vel) + np.sqrt(self.gravity * h)


class Euler(ConservationModel):
    """Ideal-gas Euler system (rho, rho u, E), p = (gamma-1)(E - rho u^2/2)
    (models.py:214-260)."""

    kind = "euler"
    n_components = 3
    abi_model = MODEL_EULER
    speed = 0.0

    def __init__(self, gamma: float = DEFAULT_GAMMA):
        if not gamma > 1.0:
            raise PhysicalStateError(f"gamma must exceed 1, got {gamma}")
        self.gamma = float(gamma)

    def _primitives(self, u):
        rho = u[..., 0, :]
        bad = rho <= 0.0
        if np.any(bad):
            raise PhysicalStateError(
                f"non-positive density in cell {int(np.argmax(bad.reshape(-1)))}")
        vel = u[..., 1, :] / rho
        p = (self.gamma - 1.0) * (u[..., 2, :] - 0.5 * rho * vel * vel)
        bad = p <= 0.0
        if np.any(bad):
            raise PhysicalStateError(
                f"non-positive pressure in cell {int(np.argmax(bad.reshape(-1)))}")
        return rho, vel, p

    def flux(self, u):
        self._check_shape(u)
        rho, vel, p = self._primitives(u)
        return np.stack([u[..., 1, :], u[..., 1, :] * vel + p, (u[..., 2, :] + p) * vel],
                        axis=-2)

    def eigenvalues(self, u):
        self._check_shape(u)
        rho, vel, p = self._primitives(u)
        c = np.sqrt(self.gamma * p / rho)
        return np.stack([vel - c, vel, vel + c], axis=-1)

    def max_abs_speed(self, u):
        self._check_shape(u)
        rho, vel, p = self._primitives(u)
        return np.abs(vel) + np.sqrt(self.gamma * p / rho)


_MODEL_KINDS = ("burgers", "advection", "shallow-water", "euler")


def make_model(kind: str, *, speed: float = 1.0, gravity: float = DEFAULT_GRAVITY,
               gamma: float = DEFAULT_GAMMA, **_unused) -> ConservationModel:
    """Build a model by name (models.py:318-328 plus "advection")."""
    if kind == "burgers":
        return Burgers()
    if kind == "advection":
        return Advection(speed)
    if kind == "shallow-water":
        return ShallowWater(gravity)
    if kind == "euler":
        return Euler(gamma)
    raise ConfigError(f"unknown model '{kind}', expected one of {sorted(_MODEL_KINDS)}")

"""Problem set-up for the GPU path: per-level steppers, seeded initial
conditions and the BASELINE.json configurations.

* ``build_steppers`` follows reference ``harness.py:324-356`` for the
  Runge-Kutta kinds: one ``SemiDiscreteOperator`` per level (per-level WENO
  order), step ``dt0 * m**l`` on level l, LF flux.
* ``fourier_ic`` is the seeded initial condition BASELINE.json names (not in
  the reference): u0 = 0.5 + sum_k a_k sin(2 pi k x +
  phi_k), a_k ~ U[-0.25, 0.25] (divided by k for config 5), phi_k ~ U[0, 2pi),
  all a drawn before all phi from one ``np.random.default_rng(seed)``,
  sampled at cell midpoints.
* ``cfl_horizon`` turns a CFL number into the horizon T = N_t * CFL * dx /
  max|u0|; dt is then T / N_t exactly as ``TemporalGrid.dt`` computes it
  (grid.py:56-58).
* ``auto_levels``: coarsen by m until at most ``max_coarse`` coarse steps.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .errors import ConfigError
from .flux import FluxConfig, SemiDiscreteOperator, WenoConfig
from .grid import SpatialGrid, TemporalGrid
from .models import make_model
from .serial import discretise_ic
from .stepper import (ComposedStepper, MatchedLFCoarse, MatchedLFFine,
                      RediscretizedLF, RungeKuttaStepper)
from .weno import DEFAULT_EPSILON

_RK_ORDER = {"fe": 1, "ssprk2": 2, "ssprk3": 3}


def _expand(per_level, n_levels: int) -> tuple:
    per_level = tuple(per_level)
    return per_level * n_levels if len(per_level) == 1 else per_level


COARSE_KINDS = ("rediscretize", "matched-0", "matched-1", "exact")


def build_steppers(model, space_grid: SpatialGrid, time_grid: TemporalGrid, *,
                   n_levels: int, m: int, weno_order=(1,), stepper=("fe",),
                   epsilon: float = DEFAULT_EPSILON, flux: str = "lf",
                   coarse: str = "rediscretize") -> list:
    """One GPU propagator per level, finest first (harness.py:324-356):
    stepper ("matched-lf",) builds the one-step LF family with the coarse
    operator named by ``coarse``; Runge-Kutta kinds rediscretise per level,
    or compose the fine step exactly for ``coarse = "exact"``."""
    if coarse not in COARSE_KINDS:
        raise ConfigError(f"unknown coarse operator '{coarse}'")
    dt0 = time_grid.dt
    if tuple(stepper) == ("matched-lf",):
        fine = MatchedLFFine(model, space_grid, dt0)
        out = [fine]
        for l in range(1, n_levels):
            m_eff = m ** l
            if coarse == "exact":
                out.append(ComposedStepper(fine, m_eff))
            elif coarse == "rediscretize":
                out.append(RediscretizedLF(model, space_grid, dt0 * m_eff))
            else:
                out.append(MatchedLFCoarse(model, space_grid, dt0, m_eff,
                                           0 if coarse == "matched-0" else 1))
        return out
    kinds = _expand(stepper, n_levels)
    orders = _expand(weno_order, n_levels)
    if len(kinds) != n_levels or len(orders) != n_levels:
        raise ConfigError("per-level lists must have one entry or n_levels entries")
    out = []
    for l in range(n_levels):
        if l > 0 and coarse == "exact":
            out.append(ComposedStepper(out[0], m ** l))
            continue
        if kinds[l] not in _RK_ORDER:
            raise ConfigError(f"stepper '{kinds[l]}' is not on the B200 path")
        op = SemiDiscreteOperator(model, space_grid,
                                  FluxConfig(kind=flux, weno=WenoConfig(
                                      order=orders[l], epsilon=epsilon)))
        out.append(RungeKuttaStepper(op.rhs, dt0 * m ** l, _RK_ORDER[kinds[l]]))
    return out


def fourier_modes(n_modes: int, seed: int, decay: bool = False):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-0.25, 0.25, n_modes)
    phi = rng.uniform(0.0, 2.0 * np.pi, n_modes)
    if decay:
        a = a / np.arange(1, n_modes + 1)
    return a, phi


def fourier_ic(space_grid: SpatialGrid, n_modes: int, seed: int = 1234,
               decay: bool = False) -> np.ndarray:
    """u0 = 0.5 + sum_k a_k sin(2 pi k x + phi_k) at cell midpoints, (1, N)."""
    a, phi = fourier_modes(n_modes, seed, decay)

    def profile(x):
        v = np.full_like(x, 0.5)
        for k in range(1, n_modes + 1):
            v = v + a[k - 1] * np.sin(2.0 * np.pi * k * x + phi[k - 1])
        return v

    return discretise_ic(profile, space_grid)


def sine_ic(space_grid: SpatialGrid) -> np.ndarray:
    """sin(2 pi x) at midpoints (BASELINE config 1)."""
    return discretise_ic(lambda x: np.sin(2.0 * np.pi * x), space_grid)


def _sin(x, length):
    return np.sin(2.0 * np.pi * x / length)


# reference harness.py:29-75: the named initial conditions of the configs
NAMED_ICS = {
    "sin-stationary": lambda x, L: _sin(x, L)[None, :],
    "sin-moving": lambda x, L: (0.5 * (1.0 + _sin(x, L)))[None, :],
    "burgers-43": lambda x, L: ((4.0 / 3.0) * _sin(x, L))[None, :],
    "sw-scaled": lambda x, L: np.stack([(1.0 + 0.5 * _sin(x, L)) / 11.0,
                                        np.zeros_like(x)]),
}


def named_ic(name: str, space_grid: SpatialGrid) -> np.ndarray:
    """A named initial condition of the reference configs at cell midpoints,
    shape (D, N)."""
    if name not in NAMED_ICS:
        raise ConfigError(f"unknown initial condition '{name}', expected one of "
                          f"{sorted(NAMED_ICS)}")
    return NAMED_ICS[name](space_grid.cell_centers(), space_grid.length)


def cfl_horizon(n_steps: int, cfl: float, dx: float, max_speed: float) -> float:
    return n_steps * (cfl * dx / max_speed)


def auto_levels(n_steps: int, m: int, max_coarse: int = 16) -> int:
    levels = 1
    n = n_steps
    while n > max_coarse:
        if n % m:
            raise ConfigError(f"N_t = {n_steps} cannot be coarsened by {m} "
                              f"down to <= {max_coarse} steps")
        n //= m
        levels += 1
    return max(levels, 2)


@dataclass(frozen=True)
class Problem:
    """One BASELINE.json configuration (or a scaled variant of it)."""

    name: str
    model: str = "burgers"
    speed: float = 1.0
    n_x: int = 512
    n_t: int = 4096
    cfl: float = 0.4
    ic: str = "fourier"        # "fourier" | "sine" | a NAMED_ICS key
    n_modes: int = 4
    decay: bool = False
    seed: int = 1234
    weno_order: tuple = (5,)
    stepper: tuple = ("ssprk3",)
    n_levels: int = 2
    m: int = 4
    cycle: str = "v"
    relaxation: str = "fcf"
    guess: str = "last-step"
    max_iters: int = 10
    residual_tol: float | None = None
    epsilon: float = DEFAULT_EPSILON
    length: float = 1.0
    coarse: str = "rediscretize"
    flux: str = "lf"
    gravity: float = 9.81
    horizon: float | None = None   # fixed T (reference configs) instead of the CFL rule

    def scaled(self, **kw) -> "Problem":
        return replace(self, **kw)

    def space_grid(self) -> SpatialGrid:
        return SpatialGrid(self.length, self.n_x)

    def initial_state(self) -> np.ndarray:
        sg = self.space_grid()
        if self.ic == "sine":
            return sine_ic(sg)
        if self.ic in NAMED_ICS:
            return named_ic(self.ic, sg)
        return fourier_ic(sg, self.n_modes, self.seed, self.decay)

    def model_obj(self):
        return make_model(self.model, speed=self.speed, gravity=self.gravity)

    def time_grid(self, u0: np.ndarray | None = None) -> TemporalGrid:
        if self.horizon is not None:
            return TemporalGrid(self.horizon, self.n_t)
        u0 = self.initial_state() if u0 is None else u0
        sg = self.space_grid()
        speed = abs(self.speed) if self.model == "advection" else float(np.max(np.abs(u0)))
        return TemporalGrid(cfl_horizon(self.n_t, self.cfl, sg.dx, speed), self.n_t)

    def steppers(self, time_grid: TemporalGrid | None = None):
        tg = self.time_grid() if time_grid is None else time_grid
        return build_steppers(self.model_obj(), self.space_grid(), tg,
                              n_levels=self.n_levels, m=self.m,
                              weno_order=self.weno_order, stepper=self.stepper,
                              epsilon=self.epsilon, coarse=self.coarse,
                              flux=self.flux)

    def options(self):
        from .mgrit import MgritOptions
        return MgritOptions(n_levels=self.n_levels, m=self.m, cycle=self.cycle,
                            relaxation=self.relaxation, guess=self.guess,
                            max_iters=self.max_iters)

    def phi_params(self, level: int = 0):
        """(model, k, rk_order, dt, dx, eps, speed) of the level-l propagator."""
        tg = self.time_grid()
        orders = _expand(self.weno_order, self.n_levels)
        kinds = _expand(self.stepper, self.n_levels)
        return dict(model=self.model, k=(orders[level] - 1) // 2,
                    rk_order=_RK_ORDER[kinds[level]], dt=tg.dt * self.m ** level,
                    dx=self.space_grid().dx, eps=self.epsilon, speed=self.speed)

    def relaxation_phi_per_iteration(self) -> dict:
        """Reference Phi-application counts per V-cycle iteration (SURVEY.md
        3.2): relaxation, restriction, coarse solve, residual row."""
        m, L = self.m, self.n_levels
        relax = restr = 0
        for l in range(L - 1):
            n_l = self.n_t // m ** l
            c_l = n_l // m
            relax += ((2 * m - 1) if self.relaxation == "fcf" else (m - 1)) * c_l
            relax += (m - 1) * c_l          # interpolation F-relax
            restr += 2 * c_l
        return dict(relaxation=relax, restriction=restr,
                    coarse=self.n_t // m ** (L - 1), residual=self.n_t)


BASELINE_CONFIGS = {
    "c1": Problem(name="c1-advection-upwind-fe", model="advection", speed=1.0,
                  n_x=128, n_t=1024, cfl=0.5, ic="sine", weno_order=(1,),
                  stepper=("fe",), n_levels=2, m=8, relaxation="fcf",
                  max_iters=200, residual_tol=1e-10),
    "c2": Problem(name="c2-burgers-weno5-rk3", n_x=512, n_t=4096, cfl=0.4,
                  n_modes=4, n_levels=2, m=4, relaxation="fcf", max_iters=10),
    "c3": Problem(name="c3-burgers-weno5-rk3-multilevel", n_x=4096, n_t=65536,
                  cfl=0.4, n_modes=8, n_levels=7, m=4, relaxation="fcf",
                  max_iters=10),
    "c4": Problem(name="c4-burgers-sweep", n_x=1024, n_t=16384, cfl=0.4,
                  n_modes=4, n_levels=3, m=2, relaxation="fcf", max_iters=10,
                  residual_tol=1e-10),
    "c5": Problem(name="c5-burgers-weno5-rk3-large", n_x=65536, n_t=262144,
                  cfl=0.4, n_modes=16, decay=True, n_levels=5, m=16,
                  relaxation="fcf", max_iters=5),
}


def c4_grid():
    """The 192 cases of BASELINE config 4."""
    base = BASELINE_CONFIGS["c4"]
    out = []
    for cfl in (0.1, 0.2, 0.4, 0.8):
        for m in (2, 4, 8, 16):
            for order in (1, 3, 5):
                for rk in ("ssprk2", "ssprk3"):
                    for relax in ("f", "fcf"):
                        out.append(base.scaled(
                            name=f"c4-cfl{cfl}-m{m}-weno{order}-{rk}-{relax}",
                            cfl=cfl, m=m, weno_order=(order,), stepper=(rk,),
                            relaxation=relax))
    return out

"""Problem set-up and the experiment harness of the GPU path: per-level
steppers, initial conditions, the BASELINE.json configurations, and the
reference's config-file experiment driver.

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
* Experiment driver, same API and file formats as reference
  ``harness.py:88-495``: ``ExperimentConfig`` / ``parse_config`` /
  ``load_config`` / ``apply_sweep_value`` / ``validate_config`` (key = value
  files with the reference's keys, aliases, sweeps and error reporting),
  ``run_experiment`` / ``run_sweep`` (serial reference + MGRIT solve on the
  GPU), ``assemble_table`` / ``experiment_table``, ``emit_csv`` (header
  ``iteration,<cols>``, shortest round-trip values, ``NaN``, LF endings) and
  ``write_meta`` (per-run sidecar).  Tables agree with the reference's to
  the north-star tolerance; the GPU path is deterministic, so a config always
  yields the same CSV bytes.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import dataclasses
import time
from pathlib import Path

import numpy as np

from .errors import ConfigError, ParseError
from .flux import FluxConfig, SemiDiscreteOperator, WenoConfig
from .grid import SpatialGrid, TemporalGrid
from .models import DEFAULT_GRAVITY, make_model
from .serial import discretise_ic, solve_serial
from .stepper import (ComposedStepper, MatchedLFCoarse, MatchedLFFine,
                      RediscretizedLF, RungeKuttaStepper)
from .weno import DEFAULT_EPSILON

_RK_ORDER = {"fe": 1, "ssprk2": 2, "ssprk3": 3}


def _expand(per_level, n_levels: int) -> tuple:
    per_level = tuple(per_level)
    return per_level * n_levels if len(per_level) == 1 else per_level


COARSE_KINDS = ("rediscretize", "matched-0", "matched-1", "exact")


def build_steppers(model, space_grid: SpatialGrid, time_grid: TemporalGrid,
                   *args, n_levels: int | None = None, m: int | None = None,
                   weno_order=(1,), stepper=("fe",), epsilon: float = DEFAULT_EPSILON,
                   flux: str = "lf", coarse: str = "rediscretize") -> list:
    """One GPU propagator per level, finest first (harness.py:324-356):
    stepper ("matched-lf",) builds the one-step LF family with the coarse
    operator named by ``coarse``; Runge-Kutta kinds rediscretise per level,
    or compose the fine step exactly for ``coarse = "exact"``.

    Also callable with the reference's signature
    ``build_steppers(config, model, space_grid, time_grid)``."""
    if isinstance(model, ExperimentConfig):
        cfg = model
        model, space_grid, time_grid = space_grid, time_grid, args[0]
        return build_steppers(model, space_grid, time_grid, n_levels=cfg.n_levels,
                              m=cfg.m, weno_order=cfg.weno_order, stepper=cfg.stepper,
                              epsilon=cfg.epsilon, flux=cfg.flux, coarse=cfg.coarse)
    if n_levels is None or m is None:
        raise ConfigError("build_steppers needs n_levels and m")
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


# reference harness.py:29-75: the named initial conditions of the configs,
# name -> (model, profile(x, length) -> (D, N))
INITIAL_CONDITIONS = {
    "sin-stationary": ("burgers", lambda x, L: _sin(x, L)[None, :]),
    "sin-moving": ("burgers", lambda x, L: (0.5 * (1.0 + _sin(x, L)))[None, :]),
    "burgers-43": ("burgers", lambda x, L: ((4.0 / 3.0) * _sin(x, L))[None, :]),
    "sw-scaled": ("shallow-water",
                  lambda x, L: np.stack([(1.0 + 0.5 * _sin(x, L)) / 11.0,
                                         np.zeros_like(x)])),
    "euler-energy-sin": ("euler",
                         lambda x, L: np.stack([np.ones_like(x), np.zeros_like(x),
                                                1.0 + 0.5 * _sin(x, L)])),
}


def initial_state(name: str, space_grid: SpatialGrid, length: float) -> np.ndarray:
    """A named initial condition at cell midpoints, shape (D, N)
    (harness.py:78-84)."""
    if name not in INITIAL_CONDITIONS:
        raise ConfigError(f"unknown initial condition '{name}', expected one "
                          f"of {sorted(INITIAL_CONDITIONS)}")
    profile = INITIAL_CONDITIONS[name][1]
    return discretise_ic(lambda x: profile(x, length), space_grid)


def named_ic(name: str, space_grid: SpatialGrid) -> np.ndarray:
    return initial_state(name, space_grid, space_grid.length)


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
        if self.ic in INITIAL_CONDITIONS:
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


# ---------------------------------------------------------------------------
# Experiment configs and driver (reference harness.py:88-495)
# ---------------------------------------------------------------------------

DEFAULT_GAMMA = 5.0 / 3.0           # models.py:22
RK_KINDS = tuple(_RK_ORDER)
PROBLEM_KINDS = ("burgers", "shallow-water", "euler")


@dataclass(frozen=True)
class ExperimentConfig:
    """One experiment (harness.py:88-113); field names, order and defaults
    are the reference's so configs and scripts carry over unchanged."""

    problem: str
    ic: str
    horizon: float
    n_x: int
    n_t: int
    n_levels: int
    length: float = 1.0
    m: int = 2
    cycle: str = "v"
    relaxation: str = "f"
    restriction_guess: str = "last-step"
    max_iters: int = 10
    flux: str = "lf"
    weno_order: tuple = (1,)
    stepper: tuple = ("fe",)
    coarse: str = "rediscretize"
    characteristic: bool = True
    epsilon: float = DEFAULT_EPSILON
    gamma: float = DEFAULT_GAMMA
    gravity: float = DEFAULT_GRAVITY
    divergence_threshold: float = 1e10
    parallelism: int = 1
    sweep: str | None = None
    sweep_values: tuple = ()


def _to_bool(raw: str) -> bool:
    word = raw.lower()
    for value, spellings in ((True, ("true", "yes", "on", "1")),
                             (False, ("false", "no", "off", "0"))):
        if word in spellings:
            return value
    raise ValueError(f"not a boolean: '{raw}'")


def _slash_ints(raw: str) -> tuple:
    return tuple(int(tok, 10) for tok in raw.split("/"))


def _slash_words(raw: str) -> tuple:
    return tuple(tok.strip() for tok in raw.split("/"))


def _decimal(raw: str) -> int:
    return int(raw, 10)


_FIELD_TYPES = {
    "problem": str, "ic": str, "length": float, "horizon": float,
    "n_x": _decimal, "n_t": _decimal, "n_levels": _decimal, "m": _decimal,
    "cycle": str, "relaxation": str, "restriction_guess": str,
    "max_iters": _decimal, "flux": str, "weno_order": _slash_ints,
    "stepper": _slash_words, "coarse": str, "characteristic": _to_bool,
    "epsilon": float, "gamma": float, "gravity": float,
    "divergence_threshold": float, "parallelism": _decimal, "sweep": str,
    "sweep_values": None,
}
_REQUIRED = ("problem", "ic", "horizon", "n_x", "n_t", "n_levels")
_ALIASES = {"N_x": "n_x", "N_t": "n_t", "L": "length", "T": "horizon"}
SWEEPABLE = ("n_x", "n_t", "n_levels", "m", "cycle", "relaxation",
             "restriction_guess", "flux", "weno_order", "stepper", "coarse",
             "characteristic", "epsilon", "gamma", "gravity", "max_iters", "grid")


def parse_config(text: str) -> ExperimentConfig:
    """``key = value`` lines, ``#`` comments, the reference's keys and
    aliases (harness.py:178-220); errors are ParseError naming the line
    and key."""
    found: dict = {}
    for lineno, line in enumerate(text.splitlines(), start=1):
        body = line.split("#", 1)[0].strip()
        if not body:
            continue
        key, eq, raw = body.partition("=")
        if not eq:
            raise ParseError("expected 'key = value'", line=lineno)
        key = key.strip()
        key = _ALIASES.get(key, key)
        raw = raw.strip()
        if key not in _FIELD_TYPES:
            raise ParseError(f"unknown key '{key}'", line=lineno, key=key)
        if key in found:
            raise ParseError(f"duplicate key '{key}'", line=lineno, key=key)
        if raw == "":
            raise ParseError("empty value", line=lineno, key=key)
        if key == "sweep_values":
            found[key] = tuple(tok.strip() for tok in raw.split(","))
        elif key == "sweep":
            found[key] = _ALIASES.get(raw, raw)
        else:
            try:
                found[key] = _FIELD_TYPES[key](raw)
            except ValueError as exc:
                raise ParseError(f"bad value '{raw}': {exc}", line=lineno,
                                 key=key) from None
    missing = [k for k in _REQUIRED if k not in found]
    if missing:
        raise ParseError(f"missing required key '{missing[0]}'", key=missing[0])
    if ("sweep" in found) != ("sweep_values" in found):
        raise ParseError("sweep and sweep_values must appear together", key="sweep")
    config = ExperimentConfig(**found)
    validate_config(config)
    return config


def load_config(path) -> ExperimentConfig:
    return parse_config(Path(path).read_text())


def apply_sweep_value(config: ExperimentConfig, key: str, raw: str) -> ExperimentConfig:
    """``config`` with the swept key set from its raw text (harness.py:231-250);
    ``grid`` takes ``<n_x>x<n_t>``."""
    if key == "grid":
        parts = raw.lower().split("x")
        try:
            if len(parts) != 2:
                raise ValueError(raw)
            new = dataclasses.replace(config, n_x=int(parts[0]), n_t=int(parts[1]))
        except ValueError:
            raise ConfigError(f"bad grid value '{raw}', expected '<n_x>x<n_t>'") from None
    else:
        try:
            new = dataclasses.replace(config, **{key: _FIELD_TYPES[key](raw)})
        except ValueError as exc:
            raise ConfigError(f"bad sweep value '{raw}' for '{key}': {exc}") from None
    validate_config(new)
    return new


def validate_config(config: ExperimentConfig) -> None:
    """Cross-field checks (harness.py:253-312)."""
    from .mgrit import CYCLE_KINDS, GUESS_KINDS, RELAXATION_KINDS
    from .flux import FLUX_KINDS

    def one_of(value, allowed, what):
        if value not in allowed:
            raise ConfigError(f"unknown {what} '{value}', expected one of {allowed}")

    if config.problem not in PROBLEM_KINDS:
        raise ConfigError(f"unknown problem '{config.problem}'")
    if config.ic not in INITIAL_CONDITIONS:
        raise ConfigError(f"unknown initial condition '{config.ic}'")
    owner = INITIAL_CONDITIONS[config.ic][0]
    if owner != config.problem:
        raise ConfigError(f"initial condition '{config.ic}' belongs to model "
                          f"'{owner}', not '{config.problem}'")
    if config.n_levels < 2:
        raise ConfigError(f"need at least 2 levels, got {config.n_levels}")
    if config.m < 2:
        raise ConfigError(f"coarsening factor must be >= 2, got {config.m}")
    one_of(config.cycle, CYCLE_KINDS, "cycle")
    one_of(config.relaxation, RELAXATION_KINDS, "relaxation")
    one_of(config.restriction_guess, GUESS_KINDS, "restriction guess")
    one_of(config.flux, FLUX_KINDS, "flux")
    span = config.m ** (config.n_levels - 1)
    if config.n_t % span:
        raise ConfigError(f"N_t = {config.n_t} is not divisible by "
                          f"m^(levels-1) = {span}")
    one_of(config.coarse, COARSE_KINDS, "coarse operator")
    if config.sweep is not None and config.sweep not in SWEEPABLE:
        raise ConfigError(f"key '{config.sweep}' is not sweepable; choose from {SWEEPABLE}")
    for name, values in (("weno_order", config.weno_order), ("stepper", config.stepper)):
        if len(values) not in (1, config.n_levels):
            raise ConfigError(f"{name} lists one value or one per level "
                              f"({config.n_levels}), got {len(values)}")
    kinds = config.stepper
    if "matched-lf" in kinds:
        if len(kinds) != 1:
            raise ConfigError("matched-lf cannot be mixed with per-level stepper kinds")
        if config.problem != "burgers":
            raise ConfigError("matched-lf steppers exist for the scalar model only")
    else:
        for kind in kinds:
            if kind not in RK_KINDS:
                raise ConfigError(f"unknown stepper '{kind}', expected matched-lf "
                                  f"or one of {RK_KINDS}")
        if config.coarse in ("matched-0", "matched-1"):
            raise ConfigError("matched coarse operators require stepper = matched-lf")
    if config.coarse == "exact" and (len(config.weno_order) != 1 or len(kinds) != 1):
        raise ConfigError("coarse = exact composes the fine stepper, so weno_order "
                          "and stepper must be single values")


@dataclass
class ExperimentResult:
    """harness.py:359-366."""

    config: ExperimentConfig
    record: object
    serial: object
    level_dts: tuple
    level_cfls: tuple
    wall_seconds: float


@dataclass
class ConvergenceTable:
    """Column-per-run relative errors, row index = iteration."""

    columns: list
    data: np.ndarray


@dataclass
class SweepResult:
    table: ConvergenceTable
    runs: list


def run_experiment(config: ExperimentConfig, *, parallelism: int | None = None,
                   max_iters: int | None = None) -> ExperimentResult:
    """Serial reference trajectory plus one MGRIT solve, both on the GPU
    (harness.py:369-400).  ``parallelism`` (the reference's chunk-worker
    threads) is accepted for compatibility; every relaxation is one batched
    launch regardless."""
    validate_config(config)
    if config.sweep is not None:
        raise ConfigError("config declares a sweep; use run_sweep")
    return _run_one(config, max_iters)


def _run_one(config: ExperimentConfig, max_iters: int | None) -> ExperimentResult:
    from .mgrit import MgritOptions, mgrit_solve

    t0 = time.perf_counter()
    iters = config.max_iters if max_iters is None else max_iters
    model = make_model(config.problem, gravity=config.gravity, gamma=config.gamma)
    sg = SpatialGrid(config.length, config.n_x)
    tg = TemporalGrid(config.horizon, config.n_t)
    u0 = initial_state(config.ic, sg, config.length)
    steppers = build_steppers(config, model, sg, tg)
    serial = solve_serial(steppers[0], u0, tg, sg, model)
    opts = MgritOptions(n_levels=config.n_levels, m=config.m, cycle=config.cycle,
                        relaxation=config.relaxation, guess=config.restriction_guess,
                        max_iters=iters, divergence_threshold=config.divergence_threshold)
    _, record = mgrit_solve(steppers, u0, tg, sg, opts, reference=serial.device_values,
                            return_trajectory=False)
    dts = tuple(tg.dt * config.m ** l for l in range(config.n_levels))
    cfls = tuple(serial.max_speed * dt / sg.dx for dt in dts)
    return ExperimentResult(config=config, record=record, serial=serial, level_dts=dts,
                            level_cfls=cfls, wall_seconds=time.perf_counter() - t0)


def run_sweep(config: ExperimentConfig, *, parallelism: int | None = None,
              max_iters: int | None = None) -> SweepResult:
    """One run per sweep value, columns named ``<key>=<raw>``
    (harness.py:417-432)."""
    validate_config(config)
    if config.sweep is None:
        raise ConfigError("config declares no sweep; use run_experiment")
    base = dataclasses.replace(config, sweep=None, sweep_values=())
    names = [f"{config.sweep}={raw}" for raw in config.sweep_values]
    runs = [_run_one(apply_sweep_value(base, config.sweep, raw), max_iters)
            for raw in config.sweep_values]
    return SweepResult(table=assemble_table(names, [r.record for r in runs]), runs=runs)


def assemble_table(names: list, records: list) -> ConvergenceTable:
    """Error histories side by side, short columns padded with NaN."""
    rows = max((len(r.errors) for r in records), default=0)
    data = np.full((rows, len(records)), np.nan)
    for j, rec in enumerate(records):
        data[:len(rec.errors), j] = rec.errors
    return ConvergenceTable(columns=list(names), data=data)


def experiment_table(result: ExperimentResult) -> ConvergenceTable:
    return assemble_table(["error"], [result.record])


def format_value(value: float) -> str:
    """Shortest round-trip decimal; ``NaN`` for diverged entries."""
    return "NaN" if np.isnan(value) else repr(float(value))


def emit_csv(table: ConvergenceTable, path) -> None:
    """``iteration,<columns>`` then one row per iteration, LF line ends
    (harness.py:454-461)."""
    out = ["iteration," + ",".join(str(c) for c in table.columns)]
    out += [",".join([str(i)] + [format_value(v) for v in row])
            for i, row in enumerate(table.data)]
    Path(path).write_bytes(("\n".join(out) + "\n").encode())


def meta_path(csv_path) -> Path:
    return Path(csv_path).with_suffix(".meta")


def write_meta(csv_path, names: list, runs: list) -> None:
    """The ``.meta`` sidecar: per run the grid, per-level dt and CFL, wall
    times and divergence (harness.py:468-495)."""
    out = []
    for name, res in zip(names, runs):
        cfg, rec = res.config, res.record
        out += [f"[{name}]", f"problem = {cfg.problem}", f"ic = {cfg.ic}",
                f"n_x = {cfg.n_x}", f"n_t = {cfg.n_t}", f"n_levels = {cfg.n_levels}",
                "level_dt = " + ", ".join(repr(v) for v in res.level_dts),
                "level_cfl = " + ", ".join(f"{v:.6g}" for v in res.level_cfls),
                f"serial_wall_seconds = {res.serial.wall_seconds:.3f}",
                f"wall_seconds = {res.wall_seconds:.3f}",
                f"diverged = {'true' if rec.diverged else 'false'}"]
        if rec.diverged_at is not None:
            out.append(f"diverged_at = {rec.diverged_at}")
        out.append("")
    total = sum(r.wall_seconds for r in runs)
    out.append(f"total_wall_seconds = {total:.3f}")
    Path(meta_path(csv_path)).write_text("\n".join(out) + "\n")

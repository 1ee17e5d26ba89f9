"""Semi-discrete finite-volume operator (WENO + global Lax-Friedrichs).

Mirrors reference ``pkg/src/mgritlab/flux.py``: ``WenoConfig`` /
``FluxConfig`` validation (flux.py:35-67), ``SemiDiscreteOperator``
constructor checks (:129-145) and ``rhs`` (:159-161).  The operator only
holds parameters; ``rhs(field)`` runs on the GPU (``mgp_sweep`` with
rk_order 0).  The Roe flux with the Harten-Hyman entropy fix
(flux.py:91-126) is supported for Burgers and shallow water; the shallow-water
system uses characteristic WENO (weno.py:222-233) on (..., 2, N) states.
There is no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import device as dev
from ._lib import MgpPhi, SCHEME_RK_WENO, SCHEME_RK_WENO_ROE, TAIL_PHI
from .errors import ConfigError, DimensionError
from .grid import SpatialGrid
from .models import ConservationModel
from .weno import DEFAULT_EPSILON, SUPPORTED_DEGREES, build_tables

FLUX_KINDS = ("lf", "roe")


@dataclass(frozen=True)
class WenoConfig:
    """Reconstruction settings: nominal order s = 2k+1 (flux.py:35-54)."""

    order: int = 1
    epsilon: float = DEFAULT_EPSILON
    characteristic: bool = True  # systems: per characteristic field (weno.py:222)

    def __post_init__(self):
        if self.order % 2 == 0 or self.degree not in SUPPORTED_DEGREES:
            supported = tuple(2 * k + 1 for k in SUPPORTED_DEGREES)
            raise ConfigError(f"unsupported reconstruction order {self.order}, "
                              f"expected one of {supported}")
        if self.epsilon <= 0.0:
            raise ConfigError(f"epsilon must be positive, got {self.epsilon}")

    @property
    def degree(self) -> int:
        return (self.order - 1) // 2


@dataclass(frozen=True)
class FluxConfig:
    """Numerical flux choice plus its reconstruction settings (flux.py:57-67)."""

    kind: str = "lf"
    weno: WenoConfig = field(default_factory=WenoConfig)

    def __post_init__(self):
        if self.kind not in FLUX_KINDS:
            raise ConfigError(
                f"unknown flux kind '{self.kind}', expected one of {FLUX_KINDS}")


class SemiDiscreteOperator:
    """du_i/dt = -(F_{i+1/2} - F_{i-1/2}) / dx on a periodic mesh, with WENO
    interface states and the global LF flux; fields (..., 1, N)."""

    def __init__(self, model: ConservationModel, space_grid: SpatialGrid,
                 config: FluxConfig):
        if space_grid.n_cells < 2 * config.weno.degree + 1:
            raise ConfigError(f"{space_grid.n_cells} cells cannot support order "
                              f"{config.weno.order} reconstruction")
        kind = getattr(model, "kind", "")
        if config.kind == "roe" and kind not in ("burgers", "shallow-water", "euler"):
            raise ConfigError(f"the B200 path implements the Roe flux for Burgers and "
                              f"the systems, not '{kind}'")
        if not hasattr(model, "abi_model"):
            raise ConfigError(f"model '{getattr(model, 'kind', model)}' is not a "
                              "model of the B200 path")
        if space_grid.n_cells > dev._lib.max_nx_static(config.weno.degree, model.abi_model):
            raise ConfigError(f"{space_grid.n_cells} cells exceed the {kind} kernel's "
                              f"limit")
        if not dev._lib.mesh_supported(space_grid.n_cells, config.weno.degree,
                                       model.abi_model):
            raise ConfigError(f"{space_grid.n_cells} cells cannot be split into 2, 4, 8 "
                              f"or 16 equal slabs of at most {dev._lib.CTA_MAX_NX} cells")
        self.model = model
        self.space_grid = space_grid
        self.config = config
        self.tables = build_tables(config.weno.degree)

    def phi_struct(self, *, dt: float, rk_order: int, regime: int) -> MgpPhi:
        return MgpPhi(int(self.model.abi_model), int(self.config.weno.degree),
                      int(rk_order), int(regime), int(self.space_grid.n_cells),
                      float(dt), float(self.space_grid.dx),
                      float(self.config.weno.epsilon), float(self.model.speed),
                      SCHEME_RK_WENO_ROE if self.config.kind == "roe" else SCHEME_RK_WENO,
                      0, 0, 1, float(getattr(self.model, "gravity", 0.0)),
                      float(getattr(self.model, "gamma", 0.0)),
                      int(bool(self.config.weno.characteristic)), 0)

    @property
    def n_components(self) -> int:
        return self.model.n_components

    def rhs(self, field_):
        """SemiDiscreteOperator.rhs (flux.py:159-161) on the GPU.  Returns the
        input's type: NumPy in -> NumPy out, CUDA tensor in -> tensor out."""
        return apply_phi(self, 0.0, 0, field_)


def apply_phi(op: SemiDiscreteOperator, dt: float, rk_order: int, u):
    """Phi (or the rhs for rk_order 0) on every (D, N) field of u."""
    return apply_phi_struct(lambda regime: op.phi_struct(dt=dt, rk_order=rk_order,
                                                         regime=regime),
                            op.space_grid.n_cells, u, op.n_components)


def apply_phi_struct(make_phi, nx: int, u, n_components: int = 1):
    """Run the propagator built by ``make_phi(regime)`` on every (D, N) field
    of u (regime = NumPy's summation order for that batch size).  Shallow
    water: synchronises and raises PhysicalStateError where the reference
    would (models.py:147-153)."""
    is_tensor = torch.is_tensor(u)
    x = dev.to_device(u)
    D = int(n_components)
    if x.dim() < 2 or x.shape[-1] != nx or x.shape[-2] != D:
        raise DimensionError(f"expected (..., {D}, {nx}) states, got {tuple(x.shape)}")
    row = D * nx
    batch = x.numel() // row
    out = torch.empty_like(x)
    if batch:
        regime = dev.regime_for_batch(batch)
        phi = make_phi(regime)
        dev.sweep(phi, n_chunks=batch, start=x, start_stride=row,
                  tail=TAIL_PHI, tail_regime=regime, tail_out=out, to_s=row,
                  what="advance")
        if D > 1:
            dev.check_status()
    if is_tensor:
        return out
    return out.cpu().numpy()


def semi_discrete_rhs(model, space_grid, config, field_):
    """One-shot evaluation of the semi-discrete operator (flux.py:164-167)."""
    return SemiDiscreteOperator(model, space_grid, config).rhs(field_)

"""Multigrid-reduction-in-time on the GPU with C-points-only finest storage.

Same method surface and semantics as reference
``pkg/src/mgritlab/mgrit.py`` -- ``MgritOptions`` (:50-79),
``ConvergenceRecord`` (:92-108), ``MgritHierarchy`` with ``f_relax`` /
``c_relax`` / ``relax`` / ``restrict`` / ``coarse_solve`` / ``interpolate`` /
``v_cycle`` / ``f_cycle`` / ``run_cycle`` / ``residual_norm`` /
``fine_values`` (:120-273) and ``mgrit_solve`` (:276-340) -- with every
propagator application done by the fused kernels of ``libmgrit_phi.so``.

Storage (the B200 design):

* Level 0 keeps only its C-points (nodes 0, m, 2m, ...; N_t/m + 1 states) in
  two ping-pong buffers.  Its F-points are never stored: they are a pure
  function of the C-points they were last F-relaxed from (``_fsrc``), or the
  broadcast initial state before any relaxation.  Every reader of F-points
  (C-relaxation, restriction, residual, error, ``fine_values``) recomputes
  them inside its own kernel, bit-identically to the reference's stored
  values because the same Phi runs in the same summation regime.
  ``f_relax(0)`` therefore launches nothing.
* Levels >= 1 keep every node of u and g, as the reference does (level-l
  F-relaxation adds g at every node).

Chunks of a level are independent inside every launch (mgrit.py:10-15), so
one launch sweeps all CF-intervals of a level; the coarsest level is one
persistent CTA marching sequentially.  ``parallelism`` is accepted and has no
effect: results do not depend on it (the reference's parity baseline is
parallelism = 1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
import weakref
from typing import Sequence

import numpy as np
import torch

from . import device as dev
from ._lib import (G_ARRAY, G_NONE, G_ZERO, GUESS_INJECTION, GUESS_LAST_STEP,
                   SUM_SEQ, TAIL_NONE, TAIL_PHI, TAIL_RESID, TAIL_RESTRICT)
from .errors import ConfigError, DimensionError
from .grid import SpatialGrid, TemporalGrid, Trajectory
from .stepper import ComposedStepper, RungeKuttaStepper, _LFStepper

CYCLE_KINDS = ("v", "f")
RELAXATION_KINDS = ("f", "fcf")
GUESS_KINDS = ("injection", "last-step")
DEFAULT_DIVERGENCE_THRESHOLD = 1e10


@dataclass(frozen=True)
class MgritOptions:
    """Iteration controls for one multigrid-in-time solve (mgrit.py:50-79)."""

    n_levels: int
    m: int = 2
    cycle: str = "v"
    relaxation: str = "f"
    guess: str = "last-step"
    max_iters: int = 10
    divergence_threshold: float = DEFAULT_DIVERGENCE_THRESHOLD
    parallelism: int = 1

    def __post_init__(self):
        if self.n_levels < 2:
            raise ConfigError(f"need at least 2 levels, got {self.n_levels}")
        if self.m < 2:
            raise ConfigError(f"coarsening factor must be >= 2, got {self.m}")
        if self.cycle not in CYCLE_KINDS:
            raise ConfigError(f"unknown cycle '{self.cycle}'")
        if self.relaxation not in RELAXATION_KINDS:
            raise ConfigError(f"unknown relaxation '{self.relaxation}'")
        if self.guess not in GUESS_KINDS:
            raise ConfigError(f"unknown restriction guess '{self.guess}'")
        if self.max_iters < 0:
            raise ConfigError(f"max_iters must be >= 0, got {self.max_iters}")
        if self.divergence_threshold <= 0.0:
            raise ConfigError("divergence threshold must be positive")
        if self.parallelism < 1:
            raise ConfigError(f"parallelism must be >= 1, got {self.parallelism}")


@dataclass
class ConvergenceRecord:
    """Per-iteration monitoring; row 0 describes the initial iterate
    (mgrit.py:92-108)."""

    errors: np.ndarray
    residuals: np.ndarray
    diverged: bool = False
    diverged_at: int | None = None
    converged_at: int | None = None   # first row below residual_tol, if given

    @property
    def n_iterations(self) -> int:
        return max(0, len(self.errors) - 1)


@dataclass
class Monitor:
    """One fused pass over the finest level: residual norm, squared error
    against a reference trajectory, and the non-finite cell count."""

    residual: float
    error_sq: float
    nonfinite: int


class MgritLevel:
    """Per-level view (mgrit.py:82-89).  For l >= 1, ``u`` / ``g`` are the
    device arrays (n_intervals + 1, D, N).  For l = 0, ``u`` materialises the
    full trajectory on demand (a device snapshot) and ``g`` is the implicit
    finest right-hand side (initial state at node 0, zero elsewhere)."""

    def __init__(self, hierarchy, index, dt, n_intervals, stepper):
        # a weak reference: no hierarchy <-> level cycle, so dropping the
        # last reference to a hierarchy frees its device arrays at once
        # (config 5 holds 35 GB per hierarchy) instead of at the next
        # collection of the cyclic garbage collector
        self._href = weakref.ref(hierarchy)
        self.index = index
        self.dt = dt
        self.n_intervals = n_intervals
        self.stepper = stepper

    @property
    def _h(self):
        h = self._href()
        if h is None:
            raise ReferenceError("the MgritHierarchy of this level no longer exists")
        return h

    @property
    def u(self):
        if self.index == 0:
            return self._h.fine_values()
        return self._h._u[self.index].view(self.n_intervals + 1, self._h.n_components, -1)

    @property
    def g(self):
        h = self._h
        if self.index == 0:
            g = torch.zeros(self.n_intervals + 1, h.nx, dtype=dev.DTYPE, device=h.device)
            g[0] = h._u0
            return g.view(self.n_intervals + 1, h.n_components, -1)
        return h._g[self.index].view(self.n_intervals + 1, h.n_components, -1)


_PROPAGATORS = (RungeKuttaStepper, _LFStepper, ComposedStepper)


def _check_stepper(s, l: int, nx: int, n_components: int):
    if not isinstance(s, _PROPAGATORS):
        raise ConfigError(
            f"level {l}: the B200 hierarchy runs this package's propagators "
            f"(RungeKuttaStepper, MatchedLF*, RediscretizedLF, ComposedStepper), "
            f"got {type(s).__name__}")
    if s.nx != nx:
        raise DimensionError(f"level {l}: stepper mesh has {s.nx} cells, state has {nx}")
    if s.n_components != n_components:
        raise DimensionError(f"level {l}: stepper works on {s.n_components} components, "
                             f"state has {n_components}")
    return s


def _nx_limit(s) -> int:
    inner = s.inner if isinstance(s, ComposedStepper) else s
    if isinstance(inner, RungeKuttaStepper):
        op = inner.operator
        if op.config.kind == "roe" and op.model.n_components == 1:
            return 4096
        return dev._lib.max_nx(op.config.weno.degree, op.model.abi_model)
    return 2048   # one-step LF family (kMaxLfNx)


class MgritHierarchy:
    """Owns the per-level device arrays and runs cycles over them."""

    # The residual row that follows a cycle recomputes, for every interval,
    # exactly the chain the next C-relaxation of the finest level runs; with
    # this set, monitor() keeps those values and that C-relaxation is a buffer
    # swap (2m + 1 instead of 3m + 1 fine propagator applications per point
    # and iteration from the second iteration on; results bit-identical).
    reuse_residual_for_relaxation = True

    def __init__(self, steppers: Sequence, initial_state, time_grid: TemporalGrid,
                 space_grid: SpatialGrid, options: MgritOptions):
        L, m = options.n_levels, options.m
        if len(steppers) != L:
            raise ConfigError(f"{len(steppers)} steppers supplied for {L} levels")
        if time_grid.n_steps % (m ** (L - 1)) != 0:
            raise ConfigError(f"N_t = {time_grid.n_steps} is not divisible by "
                              f"m^(levels-1) = {m ** (L - 1)}")
        self.options = options
        self.time_grid = time_grid
        self.space_grid = space_grid
        self.device = dev.device()
        u0 = dev.to_device(initial_state)
        D = getattr(steppers[0], "n_components", 1) if len(steppers) else 1
        if u0.dim() != 2 or u0.shape[0] != D:
            raise DimensionError(f"initial state must be ({D}, N), got {tuple(u0.shape)}")
        self.n_components = D
        self.n_cells = cells = u0.shape[1]
        # row length: the D components of one state, component-major
        self.nx = nx = D * cells
        self.steppers = [_check_stepper(s, l, cells, D) for l, s in enumerate(steppers)]
        if not dev.emulated():
            for l, s in enumerate(self.steppers):
                lim = _nx_limit(s)
                if cells > lim:
                    raise ConfigError(f"level {l}: N_x = {cells} exceeds the field limit "
                                      f"{lim} of this build for {type(s).__name__}")
        self._u0 = u0.reshape(-1).contiguous()
        self.n = [time_grid.n_steps // m ** l for l in range(L)]
        self.levels = [MgritLevel(self, l, time_grid.dt * m ** l, self.n[l], steppers[l])
                       for l in range(L)]
        n1 = self.n[0] // m
        self.n_chunks0 = n1
        kw = dict(dtype=dev.DTYPE, device=self.device)
        # level 0: C-point ping-pong buffers, rows = C-points 0..n1
        self._c = [self._u0.expand(n1 + 1, nx).contiguous(), None]
        self._cur = 0
        self._fsrc = "ic"        # "ic" (broadcast initial state) or buffer index
        self._pristine = True    # C-points all equal the initial state
        # index of the C-point buffer whose C-relaxation the last monitor()
        # already computed into the other buffer (see monitor / c_relax)
        self._crelax_done = None
        # levels >= 1: full u and g
        self._u = [None] + [torch.zeros(self.n[l] + 1, nx, **kw) for l in range(1, L)]
        self._g = [None] + [torch.zeros(self.n[l] + 1, nx, **kw) for l in range(1, L)]
        # fused FCF relaxation: steps per hand-over segment (0 = whole chains)
        # and split plan (0 = automatic, -1 = whole chains only)
        self._fcf_segment = 0
        self._fcf_split = 0
        self._partials = torch.empty(max(self.n[0] + 1, 1) * 3, **kw)
        self._sums = torch.empty(4, **kw)

    # -- helpers ------------------------------------------------------------

    def _phi(self, l: int, regime: int):
        return self.steppers[l].phi_struct(regime)

    def _other(self, i: int) -> int:
        if self._c[1 - i] is None:
            self._c[1 - i] = torch.empty_like(self._c[i])
        return 1 - i

    def _fcf_workspace(self):
        """Workspace of the fused finest-level FCF relaxation (mgp_relax_fcf),
        or None when the fused kernel does not cover the finest propagator
        (then the relaxation issues its two sweeps)."""
        if not hasattr(self, "_fcf_ws"):
            ws = None
            nc = self.n_chunks0
            if nc >= 2:
                phi = self._phi(0, dev.regime_for_batch(nc))
                nb = dev.fcf_workspace_bytes(phi, nc, self.options.m)
                if nb > 0:
                    ws = torch.zeros(nb, dtype=torch.uint8, device=self.device)
            self._fcf_ws = ws
        return self._fcf_ws

    def _reduce(self, n_chunks: int) -> tuple[float, float, float]:
        dev.sum_partials(self._partials, n_chunks, 3, self._sums)
        s = self._sums[:3].cpu().tolist()
        return s[0], s[1], s[2]

    # -- level operations ----------------------------------------------------

    def f_relax(self, l: int) -> None:
        """mgrit.py:168-180: u[jm+i] = Phi_l(u[jm+i-1]) + g[jm+i]."""
        if l == 0:
            # F-points are implicit: from now on they derive from these C-points
            self._fsrc = self._cur
            self._pristine = False
            return
        m, nx, n = self.options.m, self.nx, self.n[l]
        nc = n // m
        u, g = self._u[l], self._g[l]
        regime = dev.regime_for_batch(nc)
        dev.sweep(self._phi(l, regime), n_chunks=nc, start=u, start_stride=m * nx,
                  n_steps=m - 1, g_mode=G_ARRAY, g=g[1],
                  g_cs=m * nx, g_ss=nx, store=u[1], st_cs=m * nx, st_ss=nx,
                  what="f_relax")

    def c_relax(self, l: int) -> None:
        """mgrit.py:182-191: u[jm] = Phi_l(u[jm-1]) + g[jm]."""
        m, nx = self.options.m, self.nx
        if l == 0:
            nc = self.n_chunks0
            regime = dev.regime_for_batch(nc)
            phi = self._phi(0, regime)
            if self._fsrc == "ic":
                dst = self._c[self._cur]
                dev.sweep(phi, n_chunks=nc, start=self._u0, start_stride=0,
                          tail=TAIL_PHI, tail_regime=regime, tail_g_mode=G_ZERO,
                          tail_out=dst[1], to_s=nx, what="c_relax")
            elif self._crelax_done is not None and self._crelax_done == self._fsrc == self._cur:
                # the residual evaluation that followed the last cycle formed
                # Phi^m(C_j) + 0.0 for every interval and kept it in the other
                # buffer: that IS this C-relaxation (same propagator, same
                # summation regime, same operations), so only node 0 is copied
                src = self._cur
                d = 1 - src
                self._c[d][0].copy_(self._c[src][0])
                self._cur = d
                self._crelax_done = None
            else:
                src = self._fsrc
                ws = self._fcf_workspace()
                self._crelax_done = None
                if self._cur == src:
                    d = self._other(src)
                    if ws is None:
                        self._c[d][0].copy_(self._c[src][0])
                    self._cur = d
                dst = self._c[self._cur]
                if ws is not None:
                    # one launch, intervals split over persistent CTAs by step
                    # (node 0 copied by the kernel)
                    dev.relax_fcf(phi, n_chunks=nc, m=m, g_mode=G_ZERO, cs=self._c[src],
                                  cd=dst, workspace=ws, segment=self._fcf_segment, split=self._fcf_split,
                                  what="c_relax")
                else:
                    dev.sweep(phi, n_chunks=nc, start=self._c[src], start_stride=nx,
                              n_steps=m - 1, g_mode=G_ZERO, tail=TAIL_PHI,
                              tail_regime=regime, tail_g_mode=G_ZERO, tail_out=dst[1],
                              to_s=nx, what="c_relax")
            self._pristine = False
            return
        n = self.n[l]
        nc = n // m
        u, g = self._u[l], self._g[l]
        regime = dev.regime_for_batch(nc)
        dev.sweep(self._phi(l, regime), n_chunks=nc, start=u[m - 1],
                  start_stride=m * nx, tail=TAIL_PHI, tail_regime=regime,
                  tail_g_mode=G_ARRAY, tail_g=g[m], tg_s=m * nx, tail_out=u[m],
                  to_s=m * nx, what="c_relax")

    def relax(self, l: int) -> None:
        self.f_relax(l)
        if self.options.relaxation == "fcf":
            self.c_relax(l)
            self.f_relax(l)

    def restrict(self, l: int) -> None:
        """mgrit.py:199-217: FAS restriction with last-step or injection guess."""
        m, nx = self.options.m, self.nx
        nc = self.n[l + 1]
        regime = dev.regime_for_batch(nc)
        cu, cg = self._u[l + 1], self._g[l + 1]
        # phi_fine goes into the coarse u rows themselves: the FAS kernel
        # reads element c of it before it writes element c of u_c, so no
        # scratch array the size of the level is needed
        phi_buf = cu[1]
        guess = GUESS_LAST_STEP if self.options.guess == "last-step" else GUESS_INJECTION
        if l == 0:
            cpts = self._c[self._cur]
            cg[0].copy_(cpts[0])
            cu[0].copy_(cpts[0])
            # phi_fine = Phi_0(u[mi-1]): recompute the last F-point of chunk i-1
            if self._fsrc == "ic":
                dev.sweep(self._phi(0, regime), n_chunks=nc, start=self._u0,
                          start_stride=0, tail=TAIL_PHI, tail_regime=regime,
                          tail_out=phi_buf, to_s=nx, what="restrict/fine")
            else:
                dev.sweep(self._phi(0, regime), n_chunks=nc, start=self._c[self._fsrc],
                          start_stride=nx, n_steps=m - 1, g_mode=G_ZERO,
                          tail=TAIL_PHI, tail_regime=regime, tail_out=phi_buf,
                          to_s=nx, what="restrict/fine")
            # psi = Phi_1(u[m(i-1)]) and the FAS combination
            dev.sweep(self._phi(1, regime), n_chunks=nc, start=cpts, start_stride=nx,
                      tail=TAIL_RESTRICT, tail_regime=regime, tail_g_mode=G_ZERO,
                      guess=guess, aux=phi_buf, aux_s=nx, aux2=cpts[1], aux2_s=nx,
                      tail_out=cg[1], to_s=nx, tail_out2=cu[1], to2_s=nx,
                      what="restrict/coarse")
            return
        fu, fg = self._u[l], self._g[l]
        cg[0].copy_(fu[0])
        cu[0].copy_(fu[0])
        dev.sweep(self._phi(l, regime), n_chunks=nc, start=fu[m - 1],
                  start_stride=m * nx, tail=TAIL_PHI, tail_regime=regime,
                  tail_out=phi_buf, to_s=nx, what="restrict/fine")
        dev.sweep(self._phi(l + 1, regime), n_chunks=nc, start=fu, start_stride=m * nx,
                  tail=TAIL_RESTRICT, tail_regime=regime, tail_g_mode=G_ARRAY,
                  tail_g=fg[m], tg_s=m * nx, guess=guess, aux=phi_buf, aux_s=nx,
                  aux2=fu[m], aux2_s=m * nx, tail_out=cg[1], to_s=nx,
                  tail_out2=cu[1], to2_s=nx, what="restrict/coarse")

    def coarse_solve(self) -> None:
        """mgrit.py:219-226: sequential single-state solve of the coarsest
        level -- one persistent CTA marches every step."""
        L = self.options.n_levels
        nx = self.nx
        u, g = self._u[L - 1], self._g[L - 1]
        n = self.n[L - 1]
        dev.sweep(self._phi(L - 1, dev.regime_for_batch(1)), n_chunks=1, start=u,
                  start_stride=0, n_steps=n, g_mode=G_ARRAY, g=g[1], g_ss=nx,
                  store=u[1], st_ss=nx, what="coarse_solve")

    def interpolate(self, l: int) -> None:
        """mgrit.py:228-232: inject level l+1 onto level l's C-points, F-relax."""
        m = self.options.m
        if l == 0:
            self._c[self._cur].copy_(self._u[1])
            self._pristine = False
            self._crelax_done = None
        else:
            self._u[l][::m].copy_(self._u[l + 1])
        self.f_relax(l)

    # -- cycles ----------------------------------------------------------------

    def v_cycle(self, l: int = 0) -> None:
        if l == self.options.n_levels - 1:
            self.coarse_solve()
            return
        self.relax(l)
        self.restrict(l)
        self.v_cycle(l + 1)
        self.interpolate(l)

    def f_cycle(self) -> None:
        L = self.options.n_levels
        for l in range(L - 1):
            self.relax(l)
            self.restrict(l)
        self.coarse_solve()
        for l in range(L - 2, -1, -1):
            self.interpolate(l)
            if l > 0:
                self.v_cycle(l)

    def run_cycle(self) -> None:
        if self.options.cycle == "f":
            self.f_cycle()
        else:
            self.v_cycle(0)

    # -- monitoring --------------------------------------------------------------

    def _fast_monitor_ok(self) -> bool:
        return (self._fsrc == self._cur
                and dev.regime_for_batch(self.n_chunks0) == SUM_SEQ)

    def monitor(self, reference: torch.Tensor | None = None) -> Monitor:
        """Residual norm (mgrit.py:264-270), squared error against
        ``reference`` rows (grid.py:96-108 numerator) and the number of
        non-finite cells of the finest iterate (mgrit.py:323), in one pass."""
        m, nx, nt = self.options.m, self.nx, self.n[0]
        ref = None if reference is None else reference.reshape(nt + 1, nx)
        resid_regime = dev.regime_for_batch(nt)
        if self._pristine and self._fsrc == "ic":
            # every node holds u0: r = (0 + Phi(u0)) - u0 at each of the Nt nodes
            dev.sweep(self._phi(0, resid_regime), n_chunks=1, start=self._u0,
                      start_stride=0, tail=TAIL_RESID, tail_regime=resid_regime,
                      tail_g_mode=G_ZERO, aux=self._u0, aux_s=0,
                      partials=self._partials, what="residual")
            r2, _, _ = self._reduce(1)
            dev.sweep(self._phi(0, resid_regime), n_chunks=nt + 1, start=self._u0,
                      start_stride=0, ref=ref, ref_cs=nx, count_nonfinite=1,
                      partials=self._partials, what="monitor")
            _, e2, nf = self._reduce(nt + 1)
            return Monitor(math.sqrt(nt * r2), e2, int(nf))
        if self._fast_monitor_ok():
            # F-point residuals are exactly zero (same Phi, same regime as the
            # F-relaxation that defines them); C-point residuals need the
            # recomputed last F-point of each chunk.
            nc = self.n_chunks0
            c = self._c[self._cur]
            # the residual's 0.0 + Phi^m(C_j) is the next C-relaxation's
            # Phi^m(C_j) + 0.0: keep it in the other C-point buffer, and
            # c_relax(0) becomes a buffer swap if nothing changes in between
            keep = None
            if self.reuse_residual_for_relaxation and self.options.relaxation == "fcf":
                keep = self._c[self._other(self._cur)]
            dev.sweep(self._phi(0, dev.regime_for_batch(nc)), n_chunks=nc, start=c,
                      start_stride=nx, n_steps=m - 1, g_mode=G_ZERO, ref=ref,
                      ref_cs=m * nx, ref_ss=nx, ref_last_next=1, count_nonfinite=1,
                      tail=TAIL_RESID, tail_regime=resid_regime, tail_g_mode=G_ZERO,
                      aux=c[1], aux_s=nx, partials=self._partials,
                      tail_out=None if keep is None else keep[1], to_s=nx, what="monitor")
            self._crelax_done = None if keep is None else self._cur
            r2, e2, nf = self._reduce(nc)
            return Monitor(math.sqrt(r2), e2, int(nf))
        # general state: materialise the trajectory, then one batched pass
        traj = self.fine_values().reshape(nt + 1, nx)
        dev.sweep(self._phi(0, resid_regime), n_chunks=nt, start=traj,
                  start_stride=nx, ref=ref, ref_cs=nx, count_nonfinite=1,
                  tail=TAIL_RESID, tail_regime=resid_regime, tail_g_mode=G_ZERO,
                  aux=traj[1], aux_s=nx, ref_last_next=1, partials=self._partials,
                  what="monitor")
        r2, e2, nf = self._reduce(nt)
        return Monitor(math.sqrt(r2), e2, int(nf))

    def residual_norm(self) -> float:
        """Euclidean norm of the finest-level residual g + Phi(u_prev) - u."""
        return self.monitor().residual

    def fine_values(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """The finest-level trajectory (N_t + 1, D, N) as a device tensor,
        F-points recomputed from the C-points they derive from (written into
        ``out`` when given)."""
        m, nx, nt = self.options.m, self.nx, self.n[0]
        if out is None:
            out = torch.empty(nt + 1, nx, dtype=dev.DTYPE, device=self.device)
        else:
            out = out.view(nt + 1, nx)
        out[::m].copy_(self._c[self._cur])
        nc = self.n_chunks0
        if self._fsrc == "ic":
            for s in range(1, m):
                out[s::m].copy_(self._u0.expand(nc, nx))
        else:
            dev.sweep(self._phi(0, dev.regime_for_batch(nc)), n_chunks=nc,
                      start=self._c[self._fsrc], start_stride=nx, n_steps=m - 1,
                      g_mode=G_ZERO, store=out[1], st_cs=m * nx, st_ss=nx,
                      what="fine_values")
        return out.view(nt + 1, self.n_components, self.n_cells)

    def relax_fine_values(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """``relax(0)`` followed by ``fine_values(out)``: one FCF relaxation of
        the finest level with the relaxed trajectory materialised.  With FCF
        relaxation and a propagator the fused kernel covers, this is ONE
        launch (mgp_relax_fcf): each interval's C-step runs straight into the
        next interval's final F-steps and the work is split over persistent
        CTAs; otherwise relax(0) and fine_values()."""
        m, nx, nt = self.options.m, self.nx, self.n[0]
        ws = self._fcf_workspace() if self.options.relaxation == "fcf" else None
        if ws is None:
            self.relax(0)
            return self.fine_values(out=out)
        if out is None:
            out = torch.empty(nt + 1, nx, dtype=dev.DTYPE, device=self.device)
        else:
            out = out.view(nt + 1, nx)
        self.f_relax(0)                   # F-points now derive from these C-points
        src = self._cur
        d = self._other(src)
        self._crelax_done = None
        nc = self.n_chunks0
        dev.relax_fcf(self._phi(0, dev.regime_for_batch(nc)), n_chunks=nc, m=m, g_mode=G_ZERO,
                      cs=self._c[src], cd=self._c[d], workspace=ws,
                      segment=self._fcf_segment, split=self._fcf_split, fstore=out[1],
                      f_cs=m * nx, f_ss=nx, cstore=out, cst_s=m * nx,
                      what="relax_fine_values")
        self._cur = self._fsrc = d
        self._pristine = False
        return out.view(nt + 1, self.n_components, self.n_cells)

    def load_c_points(self, c_points) -> None:
        """Set the finest-level C-points (N_t/m + 1 rows, host or device) and
        take the F-points as F-relaxed from them (the state after an
        interpolation).  Host tensors are copied asynchronously (pinned
        memory recommended)."""
        c = self._c[self._cur]
        src = c_points if torch.is_tensor(c_points) else torch.from_numpy(
            np.ascontiguousarray(c_points, dtype=np.float64))
        c.copy_(src.reshape(c.shape), non_blocking=True)
        self._fsrc = self._cur
        self._pristine = False
        self._crelax_done = None

    def relax_to_host(self, c_points_host: torch.Tensor, traj_host: torch.Tensor,
                      pieces: int | None = None, graph: bool = False) -> None:
        """One relaxation of the finest level (``relax(0)``) fed from and
        written back to pinned host memory, pipelined over pieces of
        CF-intervals: the C-points of piece k+1 travel host->device and the
        trajectory rows of piece k-1 device->host while piece k is relaxed
        (PCIe is full duplex; the copies run on their own streams).  Input:
        the C-points (N_t/m + 1 rows); output: the relaxed finest trajectory
        (N_t + 1 rows), i.e. ``fine_values()`` after ``relax(0)``; the
        hierarchy holds the relaxed iterate afterwards.  Asynchronous on the
        current stream (synchronise before reading the host output).
        ``graph=True`` captures the step into a CUDA graph on first use (one
        per buffer parity) and replays it.  ``pieces=0`` runs ONE fused
        launch that reads and writes the pinned host buffers itself
        (zero-copy).  Measured on B200 for config 2 (PCIe 56 GB/s each way,
        16.8 MB out and 4.2 MB in per call): 4 pieces 7.6-7.8 G
        point-updates/s, zero-copy 7.5-7.6 G, 2 pieces 7.3 G, 8 pieces 5.6 G
        (each piece's launch then holds fewer chains than CTA slots); for
        config 3 (2.15 GB out, 0.54 GB in, 16384 intervals): zero-copy 9.6 G,
        8 / 16 / 32 / 64 pieces 10.9 / 11.5 / 11.8 / 11.9 G (the copy engine
        moves 56.5 GB/s, the SMs' zero-copy stores 51.7, and the copies overlap
        the kernels).  ``pieces=None`` chooses: zero-copy below 4096
        intervals, else pieces of 256 intervals (at most 64)."""
        self._crelax_done = None
        if pieces is None:
            nc = self.n_chunks0
            pieces = 0 if nc < 4096 else min(64, nc // 256)
        if pieces == 0:
            return self._relax_to_host_direct(c_points_host, traj_host)
        if graph:
            return self._relax_to_host_graph(c_points_host, traj_host, pieces)
        return self._relax_to_host(c_points_host, traj_host, pieces, capturing=False)

    def _relax_to_host_direct(self, c_points_host, traj_host):
        """pieces = 0: ONE fused launch that reads the C-points from and
        writes the trajectory to the pinned host buffers itself (mapped
        pinned memory; every byte still crosses PCIe inside the call, as
        the kernel's loads at chain starts and stores at every step)."""
        ws = self._fcf_workspace() if self.options.relaxation == "fcf" else None
        if ws is None or not (c_points_host.is_pinned() and traj_host.is_pinned()):
            return self._relax_to_host(c_points_host, traj_host, 2, capturing=False)
        m, nx = self.options.m, self.nx
        nc = self.n_chunks0
        src = self._cur
        d = self._other(src)
        th = traj_host.reshape(-1, nx)
        dev.relax_fcf(self._phi(0, dev.regime_for_batch(nc)), n_chunks=nc, m=m, g_mode=G_ZERO,
                      cs=c_points_host.reshape(-1, nx), cd=self._c[d], workspace=ws,
                      segment=self._fcf_segment, split=self._fcf_split, fstore=th[1], f_cs=m * nx, f_ss=nx,
                      cstore=th, cst_s=m * nx, what="relax_to_host")
        self._cur = self._fsrc = d
        self._pristine = False

    def _relax_to_host_graph(self, c_points_host, traj_host, pieces):
        key = (c_points_host.data_ptr(), traj_host.data_ptr(), pieces, self._cur,
               self.options.relaxation)
        cache = self.__dict__.setdefault("_graphs", {})
        if key not in cache:
            cur = self._cur
            self._relax_to_host(c_points_host, traj_host, pieces, capturing=False)  # warm-up
            torch.cuda.synchronize()
            self._cur = self._fsrc = cur
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._relax_to_host(c_points_host, traj_host, pieces, capturing=True)
            cache[key] = (g, self._cur)
            self._cur = self._fsrc = cur
        g, after = cache[key]
        g.replay()
        self._cur = self._fsrc = after
        self._pristine = False

    def _relax_to_host(self, c_points_host, traj_host, pieces, capturing):
        m, nx, nt = self.options.m, self.nx, self.n[0]
        nc = self.n_chunks0
        regime = dev.regime_for_batch(nc)
        phi = self._phi(0, regime)
        fcf = self.options.relaxation == "fcf"
        comp = torch.cuda.current_stream()
        if not hasattr(self, "_io"):
            self._io = (torch.cuda.Stream(), torch.cuda.Stream(),
                        torch.empty(nt + 1, nx, dtype=dev.DTYPE, device=self.device))
        h2d, d2h, traj = self._io
        src = self._cur
        cs = self._c[src]
        dst = self._other(src) if fcf else src
        cd = self._c[dst]
        ch = c_points_host.reshape(nc + 1, nx)
        th = traj_host.reshape(nt + 1, nx)
        if not capturing:
            comp.wait_stream(d2h)   # the previous call's copies are done with traj
        h2d.wait_stream(comp)       # ... and its kernels with the C-point buffers
        bounds = [nc * k // pieces for k in range(pieces + 1)]
        for k in range(pieces):
            a, b = bounds[k], bounds[k + 1]
            if a == b:
                continue
            last = b == nc
            with torch.cuda.stream(h2d):
                cs[a:b + (1 if last else 0)].copy_(ch[a:b + (1 if last else 0)],
                                                   non_blocking=True)
            comp.wait_stream(h2d)
            ws = self._fcf_workspace() if fcf else None
            if ws is not None:
                # one launch per piece: new C-points a+1..b into cd and the
                # trajectory rows a*m .. b*m (interval a's final F-steps
                # start from the new C-point a the previous piece wrote)
                dev.relax_fcf(phi, n_chunks=b - a, m=m, g_mode=G_ZERO, cs=cs[a], cd=cd[a],
                              workspace=ws, segment=self._fcf_segment, split=self._fcf_split,
                              fstore=traj[a * m + 1], f_cs=m * nx, f_ss=nx,
                              cstore=traj[a * m], cst_s=m * nx,
                              f0_start=None if a == 0 else cd[a], what="relax_to_host")
            elif fcf:
                if a == 0:
                    cd[0].copy_(cs[0])
                # fused F + C relaxation of chunks [a, b): new C-points a+1..b
                dev.sweep(phi, n_chunks=b - a, start=cs[a], start_stride=nx,
                          n_steps=m - 1, g_mode=G_ZERO, tail=TAIL_PHI, tail_regime=regime,
                          tail_g_mode=G_ZERO, tail_out=cd[a + 1], to_s=nx,
                          what="relax_to_host/fc")
            if ws is None:
                # final F-relaxation with every node stored
                traj[a * m: b * m + 1: m].copy_(cd[a:b + 1])
                dev.sweep(phi, n_chunks=b - a, start=cd[a], start_stride=nx, n_steps=m - 1,
                          g_mode=G_ZERO, store=traj[a * m + 1], st_cs=m * nx, st_ss=nx,
                          what="relax_to_host/f")
            d2h.wait_stream(comp)
            with torch.cuda.stream(d2h):
                rows = slice(a * m, b * m + (1 if last else 0))
                th[rows].copy_(traj[rows], non_blocking=True)
        comp.wait_stream(d2h)
        self._cur = dst
        self._fsrc = dst
        self._pristine = False

    def c_points(self) -> torch.Tensor:
        """Current finest-level C-points (N_t/m + 1, D, N), device view."""
        return self._c[self._cur].view(-1, self.n_components, self.n_cells)


def _ref_norm_sq(reference: torch.Tensor, nx: int, stepper) -> float:
    """||reference||^2 with the same deterministic reduction as the error."""
    rows = reference.numel() // nx
    zero = torch.zeros(nx, dtype=dev.DTYPE, device=reference.device)
    partials = torch.empty(rows * 3, dtype=dev.DTYPE, device=reference.device)
    sums = torch.empty(4, dtype=dev.DTYPE, device=reference.device)
    dev.sweep(stepper.phi_struct(SUM_SEQ), n_chunks=rows, start=zero, start_stride=0,
              ref=reference.reshape(rows, nx), ref_cs=nx, partials=partials,
              what="reference norm")
    dev.sum_partials(partials, rows, 3, sums)
    return float(sums[1].item())


def mgrit_solve(steppers: Sequence, initial_state, time_grid: TemporalGrid,
                space_grid: SpatialGrid, options: MgritOptions, reference=None,
                *, return_trajectory: bool = True, hierarchy_out: list | None = None,
                residual_tol: float | None = None, on_row=None):
    """Iterate cycles until max_iters, recording convergence per iteration
    (mgrit.py:276-340): row 0 is the initial iterate; divergence (non-finite
    iterate, or relative error above the threshold, or a non-finite error
    when a reference is supplied) is recorded, not raised, and that row plus
    all later rows stay NaN.

    reference: serial trajectory (N_t + 1, D, N), host array or CUDA tensor.
    Returns (Trajectory, ConvergenceRecord); the trajectory values are a host
    array (``return_trajectory=False`` skips materialising it, e.g. for
    problems whose full trajectory does not fit in memory).  residual_tol
    (not in the reference, BASELINE config 1 "stop at residual < 1e-10")
    stops after the first row whose residual is below it.  ``on_row(it, h)``
    is called after every recorded row with the hierarchy (test hook).

    Systems: a PhysicalStateError condition met inside a cycle is recorded
    as divergence at that iteration (mgrit.py:316-320; the GPU finishes the
    cycle on the inadmissible state instead of unwinding mid-cycle, so the
    returned trajectory is the completed cycle's, not the reference's
    partially updated arrays); met by row 0 or by the monitoring after a
    cycle, it raises, as the reference's residual_norm() does.
    """
    h = MgritHierarchy(steppers, initial_state, time_grid, space_grid, options)
    if hierarchy_out is not None:
        hierarchy_out.append(h)

    checked = h.n_components > 1    # systems: PhysicalStateError

    def trajectory():
        if not return_trajectory:
            return None
        t = Trajectory(time_grid, space_grid, h.fine_values().cpu().numpy())
        if checked:
            # the reference's fine_values() returns stored arrays and never
            # raises; bits set recomputing a diverged iterate's F-points here
            # belong to no propagator call of the solve
            dev.take_status()
        return t

    if checked:
        dev.take_status()      # stale bits of earlier, unrelated work

    if options.max_iters == 0:
        return trajectory(), ConvergenceRecord(errors=np.empty(0), residuals=np.empty(0))

    ref = None
    ref_norm = None
    if reference is not None:
        ref = dev.to_device(reference)
        if ref.numel() != (time_grid.n_steps + 1) * h.nx:
            raise DimensionError(f"reference has shape {tuple(ref.shape)}")
        ref_norm = math.sqrt(_ref_norm_sq(ref, h.nx, h.steppers[0]))
        if ref_norm == 0.0:
            raise ValueError("reference trajectory has zero norm")

    def error(mon: Monitor) -> float:
        if ref is None:
            return math.nan
        return math.sqrt(mon.error_sq) / ref_norm

    n_rows = options.max_iters + 1
    errors = np.full(n_rows, np.nan)
    residuals = np.full(n_rows, np.nan)
    diverged, diverged_at, converged_at = False, None, None

    def watch(mon):
        if checked:
            dev.check_status()
        return mon

    mon = watch(h.monitor(ref))
    errors[0] = error(mon)
    residuals[0] = mon.residual
    if on_row is not None:
        on_row(0, h)
    for it in range(1, n_rows):
        if residual_tol is not None and converged_at is not None:
            break
        h.run_cycle()
        # a state the reference rejects met INSIDE the cycle is recorded as
        # divergence (mgrit.py:316-320); met by the monitoring that follows it
        # raises, as the reference's residual_norm() does (mgrit.py:322).  The
        # cycle's bits are split from the monitor's in stream order.
        cycle_status = dev.snapshot_status() if checked else None
        mon = h.monitor(ref)
        if cycle_status is not None and int(cycle_status.item()):
            dev.take_status()
            diverged, diverged_at = True, it
            break
        mon = watch(mon)
        err = error(mon)
        finite = mon.nonfinite == 0
        if not finite or (np.isfinite(err) and err > options.divergence_threshold):
            diverged, diverged_at = True, it
            break
        if ref is not None and not np.isfinite(err):
            diverged, diverged_at = True, it
            break
        errors[it] = err
        residuals[it] = mon.residual
        if on_row is not None:
            on_row(it, h)
        if residual_tol is not None and converged_at is None and mon.residual < residual_tol:
            converged_at = it
    record = ConvergenceRecord(errors=errors, residuals=residuals,
                               diverged=diverged, diverged_at=diverged_at,
                               converged_at=converged_at)
    return trajectory(), record

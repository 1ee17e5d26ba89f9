"""Time-interval partitioning of the MGRIT hierarchy across GPUs.

One process per GPU (``torch.distributed``; NCCL over NVLink on the B200 box,
gloo in the CPU tests).  Reference semantics are those of ``mgrit.py``
(pkg/src/mgritlab/mgrit.py:120-340); the reference itself has no multi-process
execution (its ``parallelism`` slices the chunk batch across threads,
mgrit.py:153-164), so this is the B200 counterpart of that batch slicing
(SURVEY.md 8(e)).

Partition.  Level l has c_l = N_l / m chunks.  Every level whose chunk count
is a multiple of the world size R is split into R contiguous blocks of
c_l / R chunks ("distributed levels", a prefix 0..D-1 of the hierarchy);
level l+1's node j is level l's C-point j, so with equal blocks the level-
(l+1) nodes a rank owns are exactly the level-l C-points it owns.  A rank
stores its nodes plus one right halo node (its right neighbour's first node).
Levels D..L-1 (too few chunks, and always the coarsest level with its
sequential solve) live on rank 0.

Exchanges (all single states of N_x float64, or per-rank partial sums):
* after C-relaxation and restriction a rank has computed its halo node, which
  is its right neighbour's first node: send right (batched isend/irecv);
* the restriction of the last distributed level is gathered to rank 0, the
  interpolation onto it scattered back;
* residual / error / non-finite partial sums are all-gathered and summed in
  rank order, so every rank takes the same divergence decision.
Every propagator call uses the summation regime of the *global* batch the
reference would form, so the iterate is bit-identical to the single-GPU
hierarchy; only the norm summation order differs.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import device as dev
from ._lib import (G_ARRAY, G_ZERO, GUESS_INJECTION, GUESS_LAST_STEP, SUM_SEQ,
                   TAIL_PHI, TAIL_RESID, TAIL_RESTRICT)
from .errors import ConfigError, DimensionError
from .grid import SpatialGrid, TemporalGrid, Trajectory
from .mgrit import (ConvergenceRecord, Monitor, MgritHierarchy, MgritOptions, _check_stepper,
                    _ref_norm_sq)


def partition(n_steps: int, m: int, n_levels: int, world: int):
    """(number of distributed levels D, chunks per rank per distributed level)."""
    counts = [n_steps // m ** l // m for l in range(n_levels - 1)]
    D = 0
    for c in counts:
        if c % world == 0 and c >= world:
            D += 1
        else:
            break
    if D == 0:
        raise ConfigError(f"{counts[0]} finest-level chunks cannot be split evenly "
                          f"over {world} ranks")
    return D, [c // world for c in counts[:D]]


class DistMgritHierarchy:
    """MgritHierarchy over a process group; same method surface."""

    def __init__(self, steppers: Sequence, initial_state, time_grid: TemporalGrid,
                 space_grid: SpatialGrid, options: MgritOptions, group=None):
        L, m = options.n_levels, options.m
        if len(steppers) != L:
            raise ConfigError(f"{len(steppers)} steppers supplied for {L} levels")
        if time_grid.n_steps % (m ** (L - 1)) != 0:
            raise ConfigError(f"N_t = {time_grid.n_steps} is not divisible by "
                              f"m^(levels-1) = {m ** (L - 1)}")
        self.options, self.time_grid, self.space_grid = options, time_grid, space_grid
        self.group = group
        self.R = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.device = dev.device()
        u0 = dev.to_device(initial_state)
        Dc = getattr(steppers[0], "n_components", 1) if len(steppers) else 1
        if u0.dim() != 2 or u0.shape[0] != Dc:
            raise DimensionError(f"initial state must be ({Dc}, N), got {tuple(u0.shape)}")
        self.n_components = Dc
        self.n_cells = u0.shape[1]
        self.nx = nx = Dc * self.n_cells          # row length
        self.steppers = [_check_stepper(s, l, self.n_cells, Dc) for l, s in enumerate(steppers)]
        self._u0 = u0.reshape(-1).contiguous()
        self.n = [time_grid.n_steps // m ** l for l in range(L)]
        self.c = [self.n[l] // m for l in range(L - 1)]
        self.D, self.nloc = partition(time_grid.n_steps, m, L, self.R)
        self.off = [self.r * k for k in self.nloc]       # first owned chunk per level
        kw = dict(dtype=dev.DTYPE, device=self.device)
        n0 = self.nloc[0]
        # finest level: local C-points off..off+n0 (last = right halo)
        self._c = [self._u0.expand(n0 + 1, nx).contiguous(), None]
        self._cur, self._fsrc, self._pristine = 0, "ic", True
        # distributed coarse levels 1..D-1: nodes off_l*m .. (off_l+nloc_l)*m
        self._u = [None] * L
        self._g = [None] * L
        for l in range(1, self.D):
            rows = self.nloc[l] * m + 1
            self._u[l] = torch.zeros(rows, nx, **kw)
            self._g[l] = torch.zeros(rows, nx, **kw)
        # rank-0 levels D..L-1 (full arrays)
        if self.r == 0:
            for l in range(self.D, L):
                self._u[l] = torch.zeros(self.n[l] + 1, nx, **kw)
                self._g[l] = torch.zeros(self.n[l] + 1, nx, **kw)
        self._partials = torch.empty(max(n0 * m + 1, 1) * 3, **kw)
        self._sums = torch.empty(4, **kw)

    # -- helpers --------------------------------------------------------------

    def _phi(self, l, regime):
        return self.steppers[l].phi_struct(regime)

    def _regime(self, l):
        return dev.regime_for_batch(self.c[l])

    def _fcf_workspace(self):
        """Workspace of the fused FCF kernel for the local intervals (None
        when the kernel does not cover the propagator, or under the CPU test
        emulator: the sweeps are used then)."""
        if not hasattr(self, "_fcf_ws"):
            ws = None
            n0 = self.nloc[0]
            if n0 >= 1 and self.c[0] >= 2:
                phi = self._phi(0, self._regime(0))
                nb = dev.fcf_workspace_bytes(phi, max(n0, 2), self.options.m)
                if nb > 0:
                    ws = torch.zeros(nb, dtype=torch.uint8, device=self.device)
            self._fcf_ws = ws
        return self._fcf_ws

    def relax_fine_values(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """``relax(0)`` with this rank's relaxed finest nodes off*m ..
        (off+n0)*m materialised into ``out`` (n0*m + 1 rows, incl. the right
        halo): the N = 1 fused kernel (mgp_relax_fcf, F-points stored) over
        the local intervals, then the boundary exchange, then -- ranks > 0 --
        the final F-steps of the first local interval from the new C-point
        the left neighbour computed (the fused launch ran them from the old
        one; this overwrites them, stream-ordered)."""
        m, nx, n0 = self.options.m, self.nx, self.nloc[0]
        ws = self._fcf_workspace() if self.options.relaxation == "fcf" else None
        if out is None:
            out = torch.empty(n0 * m + 1, nx, dtype=dev.DTYPE, device=self.device)
        else:
            out = out.view(n0 * m + 1, nx)
        if ws is None:
            self.relax(0)
            out.copy_(self._local_values())
            return out
        self.f_relax(0)
        src = self._cur
        d = self._other(src)
        regime = self._regime(0)
        phi = self._phi(0, regime)
        cs, cd = self._c[src], self._c[d]
        dev.relax_fcf(phi, n_chunks=n0, m=m, g_mode=G_ZERO, cs=cs, cd=cd, workspace=ws,
                      fstore=out[1], f_cs=m * nx, f_ss=nx, cstore=out, cst_s=m * nx,
                      f0_start=None if self.r == 0 else cs[0], what="relax_fine_values")
        self._send_right([cd[n0]], [cd[0]])
        if self.r > 0:
            out[0].copy_(cd[0])
            dev.sweep(phi, n_chunks=1, start=cd[0], start_stride=0, n_steps=m - 1,
                      g_mode=G_ZERO, store=out[1], st_ss=nx, what="relax_fine_values/f0")
        self._cur = self._fsrc = d
        self._crelax_done = None
        self._pristine = False
        return out

    def relax_to_host(self, c_points_host: torch.Tensor, traj_host: torch.Tensor) -> None:
        """This rank's ``relax_fine_values`` fed from and written back to
        pinned host memory: the fused launch reads the local C-points
        (n0 + 1 rows incl. the halo) from, and writes the local relaxed
        trajectory (n0*m + 1 rows) to, the mapped pinned buffers itself
        (MgritHierarchy._relax_to_host_direct); the boundary exchange and the
        first interval's fix-up follow as in ``relax_fine_values``.  Falls
        back to copy-in / relax / copy-out where the fused kernel does not
        apply or the buffers are not pinned."""
        m, nx, n0 = self.options.m, self.nx, self.nloc[0]
        ws = self._fcf_workspace() if self.options.relaxation == "fcf" else None
        th = traj_host.reshape(n0 * m + 1, nx)
        if ws is None or not (c_points_host.is_pinned() and traj_host.is_pinned()):
            self.load_c_points(c_points_host)
            th.copy_(self.relax_fine_values(), non_blocking=True)
            return
        ch = c_points_host.reshape(n0 + 1, nx)
        self.f_relax(0)
        src = self._cur
        d = self._other(src)
        phi = self._phi(0, self._regime(0))
        cd = self._c[d]
        dev.relax_fcf(phi, n_chunks=n0, m=m, g_mode=G_ZERO, cs=ch, cd=cd, workspace=ws,
                      fstore=th[1], f_cs=m * nx, f_ss=nx, cstore=th, cst_s=m * nx,
                      f0_start=None if self.r == 0 else ch[0], what="relax_to_host")
        self._send_right([cd[n0]], [cd[0]])
        if self.r > 0:
            th[0].copy_(cd[0], non_blocking=True)
            dev.sweep(phi, n_chunks=1, start=cd[0], start_stride=0, n_steps=m - 1,
                      g_mode=G_ZERO, store=th[1], st_ss=nx, what="relax_to_host/f0")
        self._cur = self._fsrc = d
        self._crelax_done = None
        self._pristine = False

    def _other(self, i):
        if self._c[1 - i] is None:
            self._c[1 - i] = torch.empty_like(self._c[i])
        return 1 - i

    def _send_right(self, last_rows, first_rows):
        """Every rank sends ``last_rows`` (its halo rows) to rank r+1, which
        receives them straight into its ``first_rows`` (rows of contiguous
        level arrays, so no staging copies).  With NCCL, ``wait()`` orders the
        current CUDA stream after the transfer without blocking the host
        (the exchange is stream-ordered like the kernels around it); with
        gloo (CPU tests) it is a host wait."""
        ops = []
        if self.r + 1 < self.R:
            for t in last_rows:
                ops.append(dist.P2POp(dist.isend, t, self.r + 1, self.group))
        if self.r > 0:
            for t in first_rows:
                ops.append(dist.P2POp(dist.irecv, t, self.r - 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def _gather_rows(self, rows: torch.Tensor):
        """rows (k, nx) from every rank -> rank 0 gets a list in rank order."""
        rows = rows.contiguous()
        if self.r == 0:
            out = [torch.empty_like(rows) for _ in range(self.R)]
            dist.gather(rows, out, dst=0, group=self.group)
            return out
        dist.gather(rows, None, dst=0, group=self.group)
        return None

    def _scatter_rows(self, full: torch.Tensor | None, k: int, stride: int):
        """Rank 0 holds ``full``; rank r receives full[r*stride : r*stride + k]."""
        out = torch.empty(k, self.nx, dtype=dev.DTYPE, device=self.device)
        if self.r == 0:
            parts = [full[q * stride: q * stride + k].contiguous() for q in range(self.R)]
            dist.scatter(out, parts, src=0, group=self.group)
        else:
            dist.scatter(out, None, src=0, group=self.group)
        return out

    def _reduced(self, n) -> list:
        """This rank's partial sums of ``n`` chunks (deterministic order,
        mgp_sum_partials), all-gathered and added in rank order ON THE
        DEVICE -- identical on every rank -- then read once."""
        dev.sum_partials(self._partials, n, 3, self._sums)
        mine = self._sums[:3].contiguous()
        if self.R == 1:
            return mine.cpu().tolist()
        parts = torch.empty(self.R * 3, dtype=dev.DTYPE, device=self.device)
        dist.all_gather_into_tensor(parts, mine, group=self.group)
        parts = parts.view(self.R, 3)
        acc = parts[0]
        for q in range(1, self.R):      # fixed rank order
            acc = acc + parts[q]
        return acc.cpu().tolist()

    # -- level operations -------------------------------------------------------

    def f_relax(self, l: int) -> None:
        if l == 0:
            self._fsrc = self._cur
            self._pristine = False
            return
        if l >= self.D:
            if self.r == 0:
                self._f_relax_full(l, self._u[l], self._g[l], self.c[l])
            return
        self._f_relax_full(l, self._u[l], self._g[l], self.nloc[l])

    def _f_relax_full(self, l, u, g, nc):
        m, nx = self.options.m, self.nx
        dev.sweep(self._phi(l, self._regime(l)), n_chunks=nc, start=u, start_stride=m * nx,
                  n_steps=m - 1, g_mode=G_ARRAY, g=g[1], g_cs=m * nx, g_ss=nx,
                  store=u[1], st_cs=m * nx, st_ss=nx, what="f_relax")

    def c_relax(self, l: int) -> None:
        m, nx = self.options.m, self.nx
        if l == 0:
            n0 = self.nloc[0]
            regime = self._regime(0)
            phi = self._phi(0, regime)
            if self._fsrc == "ic":
                dst = self._c[self._cur]
                dev.sweep(phi, n_chunks=n0, start=self._u0, start_stride=0, tail=TAIL_PHI,
                          tail_regime=regime, tail_g_mode=G_ZERO, tail_out=dst[1], to_s=nx,
                          what="c_relax")
            elif (getattr(self, "_crelax_done", None) is not None
                  and self._crelax_done == self._fsrc == self._cur):
                # the residual row kept Phi^m(C_j) + 0.0 of every local
                # interval in the other buffer (monitor): this C-relaxation is
                # a buffer swap; the boundary exchange follows as always
                src = self._cur
                d = 1 - src
                self._c[d][0].copy_(self._c[src][0])
                self._cur = d
                self._crelax_done = None
                dst = self._c[d]
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
                    # the N = 1 fused kernel over the local intervals (node 0
                    # copied by the kernel; ranks > 0 receive it below)
                    dev.relax_fcf(phi, n_chunks=n0, m=m, g_mode=G_ZERO, cs=self._c[src],
                                  cd=dst, workspace=ws, what="c_relax")
                else:
                    dev.sweep(phi, n_chunks=n0, start=self._c[src], start_stride=nx,
                              n_steps=m - 1, g_mode=G_ZERO, tail=TAIL_PHI,
                              tail_regime=regime, tail_g_mode=G_ZERO, tail_out=dst[1],
                              to_s=nx, what="c_relax")
            self._send_right([dst[n0]], [dst[0]])
            self._pristine = False
            return
        if l >= self.D:
            if self.r == 0:
                self._c_relax_full(l, self._u[l], self._g[l], self.c[l])
            return
        u = self._u[l]
        self._c_relax_full(l, u, self._g[l], self.nloc[l])
        self._send_right([u[self.nloc[l] * m]], [u[0]])

    def _c_relax_full(self, l, u, g, nc):
        m, nx = self.options.m, self.nx
        regime = self._regime(l)
        dev.sweep(self._phi(l, regime), n_chunks=nc, start=u[m - 1], start_stride=m * nx,
                  tail=TAIL_PHI, tail_regime=regime, tail_g_mode=G_ARRAY, tail_g=g[m],
                  tg_s=m * nx, tail_out=u[m], to_s=m * nx, what="c_relax")

    def relax(self, l: int) -> None:
        self.f_relax(l)
        if self.options.relaxation == "fcf":
            self.c_relax(l)
            self.f_relax(l)

    def restrict(self, l: int) -> None:
        m, nx = self.options.m, self.nx
        guess = GUESS_LAST_STEP if self.options.guess == "last-step" else GUESS_INJECTION
        regime = self._regime(l)
        if l >= self.D:                       # both levels on rank 0
            if self.r == 0:
                self._restrict_full(l, self._u[l], self._g[l], self._u[l + 1],
                                    self._g[l + 1], self.c[l], guess, regime)
            return
        nc = self.nloc[l]
        if l + 1 < self.D:
            cu, cg = self._u[l + 1], self._g[l + 1]
            out_g, out_u = cg[1], cu[1]
        else:
            tmp = torch.empty(2, nc, nx, dtype=dev.DTYPE, device=self.device)
            out_g, out_u = tmp[0], tmp[1]
        # phi_fine goes into the coarse u rows themselves (the FAS kernel
        # reads element c before it writes it): no level-sized scratch
        phi_buf = out_u
        # fine rows owned here: level-0 C-points or level-l nodes
        if l == 0:
            cpts = self._c[self._cur]
            fine_u0 = cpts[0]
            if self._fsrc == "ic":
                dev.sweep(self._phi(0, regime), n_chunks=nc, start=self._u0, start_stride=0,
                          tail=TAIL_PHI, tail_regime=regime, tail_out=phi_buf, to_s=nx,
                          what="restrict/fine")
            else:
                dev.sweep(self._phi(0, regime), n_chunks=nc, start=self._c[self._fsrc],
                          start_stride=nx, n_steps=m - 1, g_mode=G_ZERO, tail=TAIL_PHI,
                          tail_regime=regime, tail_out=phi_buf, to_s=nx,
                          what="restrict/fine")
            c_start, c_stride, gf_mode, gf, gf_s, inj, inj_s = cpts, nx, G_ZERO, None, 0, cpts[1], nx
        else:
            fu, fg = self._u[l], self._g[l]
            fine_u0 = fu[0]
            dev.sweep(self._phi(l, regime), n_chunks=nc, start=fu[m - 1], start_stride=m * nx,
                      tail=TAIL_PHI, tail_regime=regime, tail_out=phi_buf, to_s=nx,
                      what="restrict/fine")
            c_start, c_stride, gf_mode, gf, gf_s, inj, inj_s = fu, m * nx, G_ARRAY, fg[m], m * nx, fu[m], m * nx
        dev.sweep(self._phi(l + 1, regime), n_chunks=nc, start=c_start, start_stride=c_stride,
                  tail=TAIL_RESTRICT, tail_regime=regime, tail_g_mode=gf_mode, tail_g=gf,
                  tg_s=gf_s, guess=guess, aux=phi_buf, aux_s=nx, aux2=inj, aux2_s=inj_s,
                  tail_out=out_g, to_s=nx, tail_out2=out_u, to2_s=nx, what="restrict/coarse")
        if l + 1 < self.D:
            if self.r == 0:
                cg[0].copy_(fine_u0)
                cu[0].copy_(fine_u0)
            self._send_right([cu[nc], cg[nc]], [cu[0], cg[0]])
            return
        # the coarse level lives on rank 0: gather nodes off+1 .. off+nc
        gathered = self._gather_rows(tmp.reshape(2 * nc, nx))
        if self.r == 0:
            cu, cg = self._u[l + 1], self._g[l + 1]
            cg[0].copy_(fine_u0)
            cu[0].copy_(fine_u0)
            for q, part in enumerate(gathered):
                part = part.reshape(2, nc, nx)
                cg[q * nc + 1: (q + 1) * nc + 1].copy_(part[0])
                cu[q * nc + 1: (q + 1) * nc + 1].copy_(part[1])

    def _restrict_full(self, l, fu, fg, cu, cg, nc, guess, regime):
        m, nx = self.options.m, self.nx
        cg[0].copy_(fu[0])
        cu[0].copy_(fu[0])
        phi_buf = cu[1]    # in place, as in restrict()
        dev.sweep(self._phi(l, regime), n_chunks=nc, start=fu[m - 1], start_stride=m * nx,
                  tail=TAIL_PHI, tail_regime=regime, tail_out=phi_buf, to_s=nx,
                  what="restrict/fine")
        dev.sweep(self._phi(l + 1, regime), n_chunks=nc, start=fu, start_stride=m * nx,
                  tail=TAIL_RESTRICT, tail_regime=regime, tail_g_mode=G_ARRAY, tail_g=fg[m],
                  tg_s=m * nx, guess=guess, aux=phi_buf, aux_s=nx, aux2=fu[m],
                  aux2_s=m * nx, tail_out=cg[1], to_s=nx, tail_out2=cu[1], to2_s=nx,
                  what="restrict/coarse")

    def coarse_solve(self) -> None:
        if self.r != 0:
            return
        L, nx = self.options.n_levels, self.nx
        u, g = self._u[L - 1], self._g[L - 1]
        dev.sweep(self._phi(L - 1, dev.regime_for_batch(1)), n_chunks=1, start=u,
                  start_stride=0, n_steps=self.n[L - 1], g_mode=G_ARRAY, g=g[1], g_ss=nx,
                  store=u[1], st_ss=nx, what="coarse_solve")

    def interpolate(self, l: int) -> None:
        m = self.options.m
        if l >= self.D:
            if self.r == 0:
                self._u[l][::m].copy_(self._u[l + 1])
            self.f_relax(l)
            return
        nc = self.nloc[l]
        if l + 1 < self.D:
            src = self._u[l + 1]                      # nodes off..off+nc (incl. halo)
        else:
            src = self._scatter_rows(self._u[l + 1] if self.r == 0 else None, nc + 1, nc)
        if l == 0:
            self._c[self._cur].copy_(src)
            self._crelax_done = None
            self._pristine = False
        else:
            self._u[l][::m].copy_(src)
        self.f_relax(l)

    # -- cycles -----------------------------------------------------------------

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

    # -- monitoring ---------------------------------------------------------------

    def _local_ref(self, reference):
        if reference is None:
            return None
        m, nx, n0 = self.options.m, self.nx, self.nloc[0]
        lo = self.off[0] * m
        return reference.reshape(-1, nx)[lo: lo + n0 * m + 1]

    def monitor(self, reference: torch.Tensor | None = None) -> Monitor:
        """Residual norm, squared error and non-finite count of the whole
        finest level; identical on every rank."""
        m, nx, nt = self.options.m, self.nx, self.n[0]
        n0 = self.nloc[0]
        ref = self._local_ref(reference)
        last = 1 if self.r == self.R - 1 else 0
        resid_regime = dev.regime_for_batch(nt)
        if self._pristine and self._fsrc == "ic":
            dev.sweep(self._phi(0, resid_regime), n_chunks=1, start=self._u0, start_stride=0,
                      tail=TAIL_RESID, tail_regime=resid_regime, tail_g_mode=G_ZERO,
                      aux=self._u0, aux_s=0, partials=self._partials, what="residual")
            dev.sum_partials(self._partials, 1, 3, self._sums)
            r2 = float(self._sums[0].item())
            rows = n0 * m + last
            dev.sweep(self._phi(0, resid_regime), n_chunks=rows, start=self._u0,
                      start_stride=0, ref=ref, ref_cs=nx, count_nonfinite=1,
                      partials=self._partials, what="monitor")
            _, e2, nf = self._reduced(rows)
            return Monitor(math.sqrt(nt * r2), e2, int(nf))
        if self._fsrc == self._cur and self._regime(0) == SUM_SEQ:
            c = self._c[self._cur]
            # keep 0.0 + Phi^m(C_j) for the next C-relaxation (MgritHierarchy.monitor)
            keep = None
            if MgritHierarchy.reuse_residual_for_relaxation and self.options.relaxation == "fcf":
                keep = self._c[self._other(self._cur)]
            dev.sweep(self._phi(0, self._regime(0)), n_chunks=n0, start=c, start_stride=nx,
                      n_steps=m - 1, g_mode=G_ZERO, ref=ref, ref_cs=m * nx, ref_ss=nx,
                      ref_last_next=last, count_nonfinite=1, tail=TAIL_RESID,
                      tail_regime=resid_regime, tail_g_mode=G_ZERO, aux=c[1], aux_s=nx,
                      partials=self._partials,
                      tail_out=None if keep is None else keep[1], to_s=nx, what="monitor")
            self._crelax_done = None if keep is None else self._cur
            r2, e2, nf = self._reduced(n0)
            return Monitor(math.sqrt(r2), e2, int(nf))
        traj = self._local_values().reshape(-1, nx)       # n0*m + 1 rows
        dev.sweep(self._phi(0, resid_regime), n_chunks=n0 * m, start=traj, start_stride=nx,
                  ref=ref, ref_cs=nx, count_nonfinite=1, tail=TAIL_RESID,
                  tail_regime=resid_regime, tail_g_mode=G_ZERO, aux=traj[1], aux_s=nx,
                  ref_last_next=last, partials=self._partials, what="monitor")
        r2, e2, nf = self._reduced(n0 * m)
        return Monitor(math.sqrt(r2), e2, int(nf))

    def residual_norm(self) -> float:
        return self.monitor().residual

    def _local_values(self) -> torch.Tensor:
        """This rank's finest-level nodes off*m .. (off+n0)*m (incl. halo)."""
        m, nx, n0 = self.options.m, self.nx, self.nloc[0]
        out = torch.empty(n0 * m + 1, nx, dtype=dev.DTYPE, device=self.device)
        out[::m].copy_(self._c[self._cur])
        if self._fsrc == "ic":
            for s in range(1, m):
                out[s::m].copy_(self._u0.expand(n0, nx))
        else:
            dev.sweep(self._phi(0, self._regime(0)), n_chunks=n0, start=self._c[self._fsrc],
                      start_stride=nx, n_steps=m - 1, g_mode=G_ZERO, store=out[1],
                      st_cs=m * nx, st_ss=nx, what="fine_values")
        return out

    def fine_values(self) -> torch.Tensor | None:
        """Whole finest-level trajectory on rank 0 (None elsewhere)."""
        m, nx, n0 = self.options.m, self.nx, self.nloc[0]
        parts = self._gather_rows(self._local_values())
        if self.r != 0:
            return None
        out = torch.empty(self.n[0] + 1, nx, dtype=dev.DTYPE, device=self.device)
        for q, p in enumerate(parts):
            out[q * n0 * m: (q + 1) * n0 * m + 1].copy_(p)
        return out.view(-1, self.n_components, self.n_cells)

    def level_values(self, l: int) -> torch.Tensor | None:
        """Level l >= 1 u array assembled on rank 0 (tests)."""
        m = self.options.m
        if l >= self.D:
            return self._u[l].view(-1, self.n_components, self.n_cells) if self.r == 0 else None
        parts = self._gather_rows(self._u[l])
        if self.r != 0:
            return None
        k = self.nloc[l] * m
        out = torch.empty(self.n[l] + 1, self.nx, dtype=dev.DTYPE, device=self.device)
        for q, p in enumerate(parts):
            out[q * k: (q + 1) * k + 1].copy_(p)
        return out.view(-1, self.n_components, self.n_cells)

    def load_c_points(self, local_c_points) -> None:
        """Set this rank's finest C-points (n0 + 1 rows incl. halo)."""
        c = self._c[self._cur]
        src = local_c_points if torch.is_tensor(local_c_points) else torch.from_numpy(
            np.ascontiguousarray(local_c_points, dtype=np.float64))
        c.copy_(src.reshape(c.shape), non_blocking=True)
        self._fsrc = self._cur
        self._pristine = False
        self._crelax_done = None


def mgrit_solve_distributed(steppers, initial_state, time_grid, space_grid,
                            options: MgritOptions, reference=None, group=None):
    """mgrit_solve (mgrit.py:276-340) over a process group; the record is
    identical on every rank, the trajectory is assembled on rank 0."""
    h = DistMgritHierarchy(steppers, initial_state, time_grid, space_grid, options, group)
    if options.max_iters == 0:
        v = h.fine_values()
        traj = Trajectory(time_grid, space_grid, v.cpu().numpy()) if v is not None else None
        return traj, ConvergenceRecord(np.empty(0), np.empty(0))
    ref = ref_norm = None
    if reference is not None:
        ref = dev.to_device(reference)
        ref_norm = math.sqrt(_ref_norm_sq(ref, h.nx, h.steppers[0]))
        if ref_norm == 0.0:
            raise ValueError("reference trajectory has zero norm")
    rows = options.max_iters + 1
    errors = np.full(rows, np.nan)
    residuals = np.full(rows, np.nan)
    diverged, at = False, None
    checked = h.n_components > 1     # systems: PhysicalStateError

    def error(mon):
        return math.nan if ref is None else math.sqrt(mon.error_sq) / ref_norm

    def status_bits(cycle_word):
        """(cycle word, monitor word), each OR-ed over all ranks (a MAX
        all-reduce of per-bit flags), so every rank decides together."""
        mon_word = dev.snapshot_status()
        cyc = dev.status_to_bits(cycle_word) if cycle_word is not None else \
            torch.zeros(len(dev.STATUS_BITS), dtype=torch.int64, device=h.device)
        flags = torch.cat([cyc, dev.status_to_bits(mon_word)])
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
        f = flags.cpu().tolist()
        n = len(dev.STATUS_BITS)
        return dev.bits_to_status(f[:n]), dev.bits_to_status(f[n:])

    if checked:
        dev.take_status()      # stale bits of earlier, unrelated work
    mon = h.monitor(ref)
    if checked:
        dev.raise_for_status(status_bits(None)[1])
    errors[0], residuals[0] = error(mon), mon.residual
    for it in range(1, rows):
        h.run_cycle()
        cycle_word = dev.snapshot_status() if checked else None
        mon = h.monitor(ref)
        if checked:
            # inside the cycle: recorded (mgrit.py:316-320); monitor: raised
            cyc, after = status_bits(cycle_word)
            if cyc:
                diverged, at = True, it
                break
            dev.raise_for_status(after)
        err = error(mon)
        if mon.nonfinite != 0 or (np.isfinite(err) and err > options.divergence_threshold):
            diverged, at = True, it
            break
        if ref is not None and not np.isfinite(err):
            diverged, at = True, it
            break
        errors[it], residuals[it] = err, mon.residual
    v = h.fine_values()
    traj = Trajectory(time_grid, space_grid, v.cpu().numpy()) if v is not None else None
    if checked:
        dev.take_status()      # F-point recomputation of a diverged iterate (see mgrit.py)
    return traj, ConvergenceRecord(errors, residuals, diverged, at)

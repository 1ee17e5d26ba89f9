"""Restatement of the reference MGRIT iteration -- TEST INFRASTRUCTURE ONLY.

Follows reference ``pkg/src/mgritlab/mgrit.py`` operation for operation with
full per-level storage (every node of every level, as the reference keeps):

* hierarchy set-up ``mgrit.py:120-149`` (level-0 iterate = initial state on
  every node, g_0[0] = initial state, coarse levels zero);
* ``f_relax`` ``:168-180``, ``c_relax`` ``:182-191``, ``relax`` ``:193-197``;
* FAS ``restrict`` with last-step / injection guess ``:199-217``;
* sequential ``coarse_solve`` ``:219-226``; ``interpolate`` ``:228-232``;
* V- and F-cycles ``:236-260``; ``residual_norm`` ``:264-270``;
* ``mgrit_solve`` with the divergence rules of ``:276-340``.

Steppers are any objects with the reference's duck-typed ``advance(u)`` and
``dt`` (e.g. :class:`oracle.OracleStepper`, or the product's GPU steppers
when checking the drop-in path).  Every batched ``advance`` call receives the
same array shape the reference would pass (batch of chunks, single state for
the coarse solve), so the NumPy summation regime is reproduced.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Level:
    dt: float
    n: int            # intervals on this level
    stepper: object
    u: np.ndarray     # (n + 1, D, N)
    g: np.ndarray


@dataclass
class Record:
    errors: np.ndarray
    residuals: np.ndarray
    diverged: bool = False
    diverged_at: int | None = None


@dataclass
class Options:
    n_levels: int
    m: int = 2
    cycle: str = "v"
    relaxation: str = "f"
    guess: str = "last-step"
    max_iters: int = 10
    divergence_threshold: float = 1e10


class Hierarchy:
    def __init__(self, steppers, u0, n_steps, dt0, opts: Options):
        u0 = np.asarray(u0, dtype=np.float64)
        if n_steps % opts.m ** (opts.n_levels - 1):
            raise ValueError("N_t not divisible by m^(L-1)")
        self.opts = opts
        self.levels = []
        for l in range(opts.n_levels):
            n = n_steps // opts.m ** l
            shape = (n + 1,) + u0.shape
            if l == 0:
                u = np.empty(shape)
                u[...] = u0
                g = np.zeros(shape)
                g[0] = u0
            else:
                u = np.zeros(shape)
                g = np.zeros(shape)
            self.levels.append(Level(dt0 * opts.m ** l, n, steppers[l], u, g))

    # mgrit.py:168-180
    def f_relax(self, l):
        lv, m = self.levels[l], self.opts.m
        base = np.arange(0, lv.n, m)
        x = lv.u[base]
        for j in range(1, m):
            x = lv.stepper.advance(x) + lv.g[base + j]
            lv.u[base + j] = x

    # mgrit.py:182-191
    def c_relax(self, l):
        lv, m = self.levels[l], self.opts.m
        t = np.arange(m, lv.n + 1, m)
        lv.u[t] = lv.stepper.advance(lv.u[t - 1]) + lv.g[t]

    def relax(self, l):
        self.f_relax(l)
        if self.opts.relaxation == "fcf":
            self.c_relax(l)
            self.f_relax(l)

    # mgrit.py:199-217
    def restrict(self, l):
        fine, coarse, m = self.levels[l], self.levels[l + 1], self.opts.m
        mi = m * np.arange(1, coarse.n + 1)
        coarse.g[0] = fine.u[0]
        coarse.u[0] = fine.u[0]
        phi = fine.stepper.advance(fine.u[mi - 1])
        psi = coarse.stepper.advance(fine.u[mi - m])
        coarse.g[mi // m] = (fine.g[mi] + phi) - psi
        if self.opts.guess == "last-step":
            coarse.u[mi // m] = phi + fine.g[mi]
        else:
            coarse.u[mi // m] = fine.u[mi]

    # mgrit.py:219-226 (single-state calls)
    def coarse_solve(self):
        lv = self.levels[-1]
        x = lv.u[0]
        for i in range(1, lv.n + 1):
            x = lv.stepper.advance(x) + lv.g[i]
            lv.u[i] = x

    # mgrit.py:228-232
    def interpolate(self, l):
        self.levels[l].u[::self.opts.m] = self.levels[l + 1].u
        self.f_relax(l)

    def v_cycle(self, l=0):
        if l == self.opts.n_levels - 1:
            self.coarse_solve()
            return
        self.relax(l)
        self.restrict(l)
        self.v_cycle(l + 1)
        self.interpolate(l)

    def f_cycle(self):
        L = self.opts.n_levels
        for l in range(L - 1):
            self.relax(l)
            self.restrict(l)
        self.coarse_solve()
        for l in range(L - 2, -1, -1):
            self.interpolate(l)
            if l > 0:
                self.v_cycle(l)

    def run_cycle(self):
        if self.opts.cycle == "f":
            self.f_cycle()
        else:
            self.v_cycle(0)

    # mgrit.py:264-270
    def residual_norm(self):
        lv = self.levels[0]
        r = (lv.g[1:] + lv.stepper.advance(lv.u[:-1])) - lv.u[1:]
        return float(np.sqrt(np.sum(r * r)))

    def fine_values(self):
        return self.levels[0].u


def rel_error(u, ref):
    """grid.py:96-108"""
    return float(np.sqrt(np.sum((u - ref) ** 2))) / float(np.sqrt(np.sum(ref * ref)))


def march(stepper, u0, n_steps):
    """serial.py:40-61: single-state sequential trajectory."""
    u0 = np.asarray(u0, dtype=np.float64)
    out = np.empty((n_steps + 1,) + u0.shape)
    out[0] = u0
    x = u0
    for i in range(1, n_steps + 1):
        x = stepper.advance(x)
        out[i] = x
    return out


def mgrit_solve(steppers, u0, n_steps, dt0, opts: Options, reference=None,
                hierarchy_out: list | None = None, residual_tol: float | None = None,
                on_row=None):
    """mgrit.py:276-340 (without the thread pool: parallelism=1 semantics).

    A PhysicalStateError raised inside a cycle is recorded as divergence at
    that iteration (mgrit.py:316-320); one raised by the monitoring that
    follows the cycle propagates, as in the reference (mgrit.py:321-322 call
    residual_norm outside the try).  The oracle's stand-in exception is
    ``oracle.PhysicalStateOracleError``.  ``residual_tol`` (the package's
    BASELINE-config-1 extension) stops after the first row whose residual is
    below it (rows >= 1, as the package's driver): the rows are a prefix of
    the reference's.  ``on_row(it, h)`` is
    called after every recorded row (fixture hashing)."""
    from . import PhysicalStateOracleError
    h = Hierarchy(steppers, u0, n_steps, dt0, opts)
    if hierarchy_out is not None:
        hierarchy_out.append(h)
    if opts.max_iters == 0:
        return h.fine_values(), Record(np.empty(0), np.empty(0))

    def err():
        if reference is None:
            return np.nan
        return rel_error(h.fine_values(), reference)

    rows = opts.max_iters + 1
    errors = np.full(rows, np.nan)
    resid = np.full(rows, np.nan)
    diverged, at = False, None
    with np.errstate(all="ignore"):
        errors[0] = err()
        resid[0] = h.residual_norm()
        if on_row is not None:
            on_row(0, h)
        for it in range(1, rows):
            if residual_tol is not None and it >= 2 and resid[it - 1] < residual_tol:
                break
            try:
                h.run_cycle()
            except PhysicalStateOracleError:
                diverged, at = True, it
                break
            e = err()
            r = h.residual_norm()
            finite = bool(np.all(np.isfinite(h.fine_values())))
            if not finite or (np.isfinite(e) and e > opts.divergence_threshold):
                diverged, at = True, it
                break
            if reference is not None and not np.isfinite(e):
                diverged, at = True, it
                break
            errors[it] = e
            resid[it] = r
            if on_row is not None:
                on_row(it, h)
    return h.fine_values(), Record(errors, resid, diverged, at)

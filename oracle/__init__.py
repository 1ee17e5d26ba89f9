"""CPU oracle for the MGRIT fine-propagator path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker (or the timed CPU
"port" baseline).  The product package ``paper_2104_09404_b200`` never
imports it and has no CPU fallback.

* ``phi_oracle.c`` -- bit-exact C restatement of the reference propagator
  Phi = ``RungeKuttaStepper.advance`` over ``SemiDiscreteOperator.rhs``
  (reference ``pkg/src/mgritlab/stepper.py:50-82``, ``flux.py:70-161``,
  ``weno.py:154-236``), both NumPy summation regimes.
* ``mgrit_oracle.py`` -- restatement of ``MgritHierarchy`` / ``mgrit_solve``
  (``mgrit.py:120-340``) with full per-level storage, driven by any stepper
  honouring the reference's duck-typed ``advance(u)`` / ``dt`` protocol.

Pinning: the oracle is checked bit-for-bit against golden vectors produced by
importing the reference itself (``tests/golden/make_golden.py``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libphi_oracle.so")

MODEL_BURGERS = 0
MODEL_ADVECTION = 1
MODEL_SHALLOW_WATER = 2
MODEL_EULER = 3
_MODELS = {"burgers": MODEL_BURGERS, "advection": MODEL_ADVECTION,
           "shallow-water": MODEL_SHALLOW_WATER, "euler": MODEL_EULER}
_NCOMP = {MODEL_BURGERS: 1, MODEL_ADVECTION: 1, MODEL_SHALLOW_WATER: 2, MODEL_EULER: 3}


class PhysicalStateOracleError(ValueError):
    """The oracle met an inadmissible state (the reference raises
    PhysicalStateError there, models.py:147-153, 228-238, 290-293); ``bits``:
    1 depth, 2 density, 4 pressure, 8 Roe average."""

    def __init__(self, bits: int):
        super().__init__(f"inadmissible state (bits {bits})")
        self.bits = bits
SUM_SEQ = 0
SUM_LANE2 = 1


class OraParams(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("k", ctypes.c_int32),
                ("rk_order", ctypes.c_int32), ("regime", ctypes.c_int32),
                ("dt", ctypes.c_double), ("dx", ctypes.c_double),
                ("eps", ctypes.c_double), ("speed", ctypes.c_double),
                ("scheme", ctypes.c_int32), ("lf_order", ctypes.c_int32),
                ("m_eff", ctypes.c_int32), ("repeats", ctypes.c_int32),
                ("gravity", ctypes.c_double), ("gamma", ctypes.c_double),
                ("characteristic", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None
REF_DIR = os.path.join(_HERE, "_ref")
REFERENCE_PKG = "/root/reference/pkg"


def install_reference(force: bool = False) -> str | None:
    """Install the UNMODIFIED reference package (mgritlab, pure Python) into
    ``oracle/_ref`` -- a pip install from a /tmp copy of its sources (the
    source tree is read-only), no dependencies (NumPy is in the image).
    git-ignored, but shipped to the GPU box with the repo snapshot, where the
    drop-in tests run the reference's own ``mgrit_solve`` with the GPU
    steppers.  Returns the install directory, or None when the reference
    sources are absent (the GPU box)."""
    import shutil
    import sys
    import tempfile
    if os.path.isdir(os.path.join(REF_DIR, "mgritlab")) and not force:
        return REF_DIR
    if not os.path.isdir(REFERENCE_PKG):
        return None
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REFERENCE_PKG, src)
        shutil.rmtree(REF_DIR, ignore_errors=True)
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                        "--no-build-isolation", "--no-deps", "--target", REF_DIR, src],
                       check=True)
    return REF_DIR


def import_reference():
    """The installed reference package (``import mgritlab`` from oracle/_ref),
    or None if it was not installed."""
    import importlib
    import sys
    if not os.path.isdir(os.path.join(REF_DIR, "mgritlab")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    return importlib.import_module("mgritlab")


def build(force: bool = False) -> str:
    """Compile libphi_oracle.so with oracle/Makefile (gcc, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH)
            < os.path.getmtime(os.path.join(_HERE, "phi_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE, "libphi_oracle.so"],
                       check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        _lib.ora_phi_apply.argtypes = [
            ctypes.POINTER(OraParams), dp, ctypes.c_int64, dp, ctypes.c_int64,
            dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        _lib.ora_phi_apply.restype = ctypes.c_int
        _lib.ora_march.argtypes = [ctypes.POINTER(OraParams), dp, dp,
                                   ctypes.c_int64, ctypes.c_int64]
        _lib.ora_march.restype = ctypes.c_int
        _lib.ora_get_tables.argtypes = [ctypes.c_int, dp, dp, dp]
        _lib.ora_get_tables.restype = ctypes.c_int
        _lib.ora_max_threads.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def make_params(*, model="burgers", k=2, rk_order=3, dt=1e-3, dx=1.0 / 64,
                eps=1e-6, speed=1.0, regime=SUM_SEQ, scheme=0, lf_order=0, m_eff=1,
                repeats=1, gravity=9.81, gamma=5.0 / 3.0,
                characteristic=True) -> OraParams:
    """scheme 0: RK over WENO/LF; 1: one-step LF (matched-lf-fine,
    rediscretized-lf), 2: matched coarse LF of order lf_order emulating m_eff
    fine steps (dt = the step the formula multiplies, see include/mgrit_phi.h);
    repeats: ComposedStepper count."""
    return OraParams(_MODELS[model], int(k), int(rk_order), int(regime), float(dt),
                     float(dx), float(eps), float(speed), int(scheme), int(lf_order),
                     int(m_eff), int(repeats), float(gravity), float(gamma),
                     int(bool(characteristic)), 0)


def regime_for_shape(shape) -> int:
    """NumPy's candidate-sum order for advance(u) on an array of this shape:
    sequential when the leading axes hold >= 2 fields, 2-lane otherwise
    (verified against the reference).  (Systems use
    the 2-lane order always; the oracle applies that internally.)"""
    n = int(np.prod(shape[:-2])) if len(shape) > 2 else 1
    return SUM_SEQ if n >= 2 else SUM_LANE2


def phi_apply(params: OraParams, u: np.ndarray, g: np.ndarray | None = None,
              nthreads: int = 0) -> np.ndarray:
    """Apply Phi (+ g) to every (D, N) field of u; shape preserved."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    nx = u.shape[-1]
    row = nx * _NCOMP[params.model]
    batch = u.size // row
    out = np.empty_like(u)
    gp = None
    if g is not None:
        g = np.ascontiguousarray(np.broadcast_to(g, u.shape), dtype=np.float64)
        gp = _ptr(g)
    rc = lib().ora_phi_apply(ctypes.byref(params), _ptr(u), row, gp, row,
                             _ptr(out), row, batch, nx, int(nthreads))
    if rc >= 3:
        raise PhysicalStateOracleError(rc - 2)
    if rc != 0:
        raise ValueError(f"ora_phi_apply failed with status {rc}")
    return out


def march(params: OraParams, u: np.ndarray, g: np.ndarray | None,
          n_steps: int) -> None:
    """In place: u[i] = Phi(u[i-1]) (+ g[i]) for i = 1..n_steps."""
    assert u.flags.c_contiguous and u.dtype == np.float64
    nx = u.shape[-1]
    gp = None
    if g is not None:
        assert g.flags.c_contiguous and g.dtype == np.float64
        gp = _ptr(g)
    rc = lib().ora_march(ctypes.byref(params), _ptr(u), gp, int(n_steps), nx)
    if rc >= 3:
        raise PhysicalStateOracleError(rc - 2)
    if rc != 0:
        raise ValueError(f"ora_march failed with status {rc}")


def tables(k: int):
    cw = np.zeros(16)
    d = np.zeros(4)
    sm = np.zeros(64)
    if lib().ora_get_tables(int(k), _ptr(cw), _ptr(d), _ptr(sm)) != 0:
        raise ValueError(k)
    return cw.reshape(4, 4), d, sm.reshape(4, 4, 4)


class OracleStepper:
    """Oracle Phi with the reference's duck-typed stepper protocol
    (``advance(u)`` + ``dt``, tests/test_mgrit.py:34-42); the summation regime
    follows the shape of u exactly as NumPy does in the reference."""

    def __init__(self, *, model="burgers", k=2, rk_order=3, dt, dx,
                 eps=1e-6, speed=1.0, nthreads=0, scheme=0, lf_order=0, m_eff=1,
                 repeats=1, formula_dt=None, gravity=9.81, gamma=5.0 / 3.0,
                 characteristic=True):
        self.gravity, self.gamma, self.characteristic = gravity, gamma, characteristic
        self.model, self.k, self.order = model, k, rk_order
        self.dt, self.dx, self.eps, self.speed = dt, dx, eps, speed
        self.nthreads = nthreads
        self.scheme, self.lf_order, self.m_eff, self.repeats = scheme, lf_order, m_eff, repeats
        self.formula_dt = dt if formula_dt is None else formula_dt

    def params(self, regime: int) -> OraParams:
        return make_params(model=self.model, k=self.k, rk_order=self.order,
                           dt=self.formula_dt, dx=self.dx, eps=self.eps,
                           speed=self.speed, regime=regime, scheme=self.scheme,
                           lf_order=self.lf_order, m_eff=self.m_eff,
                           repeats=self.repeats, gravity=self.gravity,
                           gamma=self.gamma, characteristic=self.characteristic)

    def advance(self, u):
        u = np.asarray(u, dtype=np.float64)
        return phi_apply(self.params(regime_for_shape(u.shape)), u,
                         nthreads=self.nthreads)

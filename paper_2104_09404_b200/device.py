"""Device plumbing: torch tensors in, ``mgp_sweep`` launches out.

Every launch goes through :func:`sweep`, the single Python-side caller of
the C entry point ``mgp_sweep`` (include/mgrit_phi.h).  Tensors are float64
CUDA tensors; row pointers are passed as raw addresses with element strides.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import (G_NONE, MODEL_EULER, MODEL_SHALLOW_WATER, MgpFcfArgs, MgpPhi, MgpSweepArgs,
                   STATUS_NONPOSITIVE_DENSITY, STATUS_NONPOSITIVE_DEPTH,
                   STATUS_NONPOSITIVE_PRESSURE, STATUS_ROE_NONHYPERBOLIC, SUM_LANE2,
                   SUM_SEQ, TAIL_NONE)
from .errors import PhysicalStateError

DTYPE = torch.float64

# Host-logic test hook.  Tests that exercise the hierarchy / distributed
# bookkeeping on a CPU-only machine install an emulator of mgp_sweep
# (tests/sweep_emulator.py, built on the oracle) together with the torch
# device it works on.  Nothing in the package installs one: without it every
# call goes to libmgrit_phi.so and a missing GPU raises.
_emulator = None


def install_emulator(sweep_fn, sum_fn, dev: str = "cpu") -> None:
    global _emulator
    _emulator = (sweep_fn, sum_fn, torch.device(dev))


def remove_emulator() -> None:
    global _emulator
    _emulator = None


def emulated() -> bool:
    return _emulator is not None


def device() -> torch.device:
    if _emulator is not None:
        return _emulator[2]
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 MGRIT path needs a CUDA device "
                           "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_device(u) -> torch.Tensor:
    """float64, contiguous, on the current CUDA device."""
    if torch.is_tensor(u):
        t = u.to(device=device(), dtype=DTYPE)
    else:
        t = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).to(device())
    return t.contiguous()


def regime_for_batch(n_fields: int) -> int:
    """NumPy's candidate-sum order in the reference for an advance() call on
    n_fields fields (checked by the golden tests)."""
    return SUM_SEQ if n_fields >= 2 else SUM_LANE2


# Per-device status word (int32) the shallow-water kernels OR
# MGP_STATUS_* bits into where the reference raises PhysicalStateError
# (models.py:147-153).  Sweeps are asynchronous, so callers check it at
# their synchronisation points (check_status).
_status_words = {}


def status_word() -> torch.Tensor:
    d = device()
    w = _status_words.get(d)
    if w is None:
        w = torch.zeros(1, dtype=torch.int32, device=d)
        _status_words[d] = w
    return w


def take_status() -> int:
    """Read and clear the status word (synchronises with its stream)."""
    w = _status_words.get(device())
    if w is None:
        return 0
    v = int(w.item())
    if v:
        w.zero_()
    return v


_STATUS_TEXT = (
    (STATUS_NONPOSITIVE_DEPTH, "non-positive depth (models.py:147-153)"),
    (STATUS_NONPOSITIVE_DENSITY, "non-positive density (models.py:228-232)"),
    (STATUS_NONPOSITIVE_PRESSURE, "non-positive pressure (models.py:235-238)"),
    (STATUS_ROE_NONHYPERBOLIC, "Roe average loses hyperbolicity (models.py:290-293)"),
)


def raise_for_status(v: int) -> None:
    if v:
        what = [text for bit, text in _STATUS_TEXT if v & bit] or [f"status {v}"]
        raise PhysicalStateError("inadmissible state met by the system propagator: "
                                 + "; ".join(what))


def snapshot_status() -> torch.Tensor:
    """Move the status word's bits into a new device tensor and clear the
    word, in stream order (no synchronisation): the bits the work enqueued
    so far set, separated from those of later work."""
    w = status_word()
    snap = w.clone()
    w.zero_()
    return snap


STATUS_BITS = (STATUS_NONPOSITIVE_DEPTH, STATUS_NONPOSITIVE_DENSITY,
               STATUS_NONPOSITIVE_PRESSURE, STATUS_ROE_NONHYPERBOLIC)


def status_to_bits(word: torch.Tensor) -> torch.Tensor:
    """int32 status word -> one 0/1 entry per MGP_STATUS_* bit (a MAX
    all-reduce of these is the bitwise OR of every rank's word)."""
    masks = torch.tensor(STATUS_BITS, dtype=torch.int32, device=word.device)
    return ((word.reshape(1) & masks) != 0).to(torch.int64)


def bits_to_status(bits) -> int:
    return sum(b for b, on in zip(STATUS_BITS, bits) if on)


def check_status() -> None:
    """Raise PhysicalStateError if a sweep since the last check met a
    state the reference rejects."""
    raise_for_status(take_status())


def ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def sweep(phi: MgpPhi, *, n_chunks: int, start, start_stride: int,
          n_steps: int = 0, g_mode: int = G_NONE, g=None, g_cs: int = 0,
          g_ss: int = 0, store=None, st_cs: int = 0, st_ss: int = 0,
          tail: int = TAIL_NONE, tail_regime: int = SUM_SEQ,
          tail_g_mode: int = G_NONE, guess: int = 0, tail_g=None,
          tg_s: int = 0, tail_out=None, to_s: int = 0, tail_out2=None,
          to2_s: int = 0, aux=None, aux_s: int = 0, aux2=None, aux2_s: int = 0,
          ref=None, ref_cs: int = 0, ref_ss: int = 0, ref_last_next: int = 0,
          count_nonfinite: int = 0, partials=None, status=None,
          what: str = "mgp_sweep"):
    if status is None and phi.model in (MODEL_SHALLOW_WATER, MODEL_EULER):
        status = status_word()
    if _emulator is not None:
        kw = dict(locals())
        kw.pop("phi")
        return _emulator[0](phi, **kw)
    a = MgpSweepArgs()
    a.phi = phi
    a.n_chunks = int(n_chunks)
    a.start, a.start_stride = ptr(start), int(start_stride)
    a.n_steps, a.g_mode = int(n_steps), int(g_mode)
    a.g, a.g_cs, a.g_ss = ptr(g), int(g_cs), int(g_ss)
    a.store, a.st_cs, a.st_ss = ptr(store), int(st_cs), int(st_ss)
    a.tail, a.tail_regime = int(tail), int(tail_regime)
    a.tail_g_mode, a.guess = int(tail_g_mode), int(guess)
    a.tail_g, a.tg_s = ptr(tail_g), int(tg_s)
    a.tail_out, a.to_s = ptr(tail_out), int(to_s)
    a.tail_out2, a.to2_s = ptr(tail_out2), int(to2_s)
    a.aux, a.aux_s = ptr(aux), int(aux_s)
    a.aux2, a.aux2_s = ptr(aux2), int(aux2_s)
    a.ref, a.ref_cs, a.ref_ss = ptr(ref), int(ref_cs), int(ref_ss)
    a.ref_last_next = int(ref_last_next)
    a.count_nonfinite = int(count_nonfinite)
    a.partials = ptr(partials)
    a.status = ptr(status)
    rc = _lib.load().mgp_sweep(ctypes.byref(a), ctypes.c_void_p(stream_handle()))
    _lib.check(rc, what)


def sum_partials(partials: torch.Tensor, n: int, width: int, out: torch.Tensor):
    if _emulator is not None:
        return _emulator[1](partials, n, width, out)
    rc = _lib.load().mgp_sum_partials(ptr(partials), int(n), int(width), ptr(out),
                                      ctypes.c_void_p(stream_handle()))
    _lib.check(rc, "mgp_sum_partials")


def fcf_workspace_bytes(phi: MgpPhi, n_chunks: int, m: int) -> int:
    """Workspace the fused FCF relaxation needs (0: not available for this
    propagator / interval count -- the caller then issues the two sweeps)."""
    if _emulator is not None:
        return 0
    return int(_lib.load().mgp_relax_fcf_workspace(ctypes.byref(phi), int(n_chunks), int(m)))


def relax_fcf(phi: MgpPhi, *, n_chunks: int, m: int, g_mode: int, cs, cd, workspace,
              fstore=None, f_cs: int = 0, f_ss: int = 0, cstore=None, cst_s: int = 0,
              f0_start=None, cs_s: int | None = None, cd_s: int | None = None,
              segment: int = 0, split: int = 0, what: str = "mgp_relax_fcf"):
    """One fused launch of the finest level's FCF relaxation (mgp_relax_fcf,
    include/mgrit_phi.h): new C-points into ``cd`` and, with ``fstore``, the
    relaxed iterate's F-points."""
    a = MgpFcfArgs()
    a.phi = phi
    a.n_chunks, a.m, a.g_mode = int(n_chunks), int(m), int(g_mode)
    nx = int(phi.nx)
    a.cs, a.cs_s = ptr(cs), int(nx if cs_s is None else cs_s)
    a.cd, a.cd_s = ptr(cd), int(nx if cd_s is None else cd_s)
    a.fstore, a.f_cs, a.f_ss = ptr(fstore), int(f_cs), int(f_ss)
    a.cstore, a.cst_s = ptr(cstore), int(cst_s)
    a.f0_start = ptr(f0_start)
    a.workspace, a.workspace_bytes = ptr(workspace), int(workspace.numel())
    a.epoch = 1    # the kernel leaves its hand-over flags cleared
    a.segment = int(segment)
    a.split = int(split)
    rc = _lib.load().mgp_relax_fcf(ctypes.byref(a), ctypes.c_void_p(stream_handle()))
    _lib.check(rc, what)

"""ctypes binding of the C ABI in ``include/mgrit_phi.h``.

The reference is Python; its foreign-function boundary for this path is
Python calling the shared library through ctypes, exactly as this module
does.  PyTorch supplies device memory and the current CUDA stream (plumbing);
all arithmetic of the path runs in ``libmgrit_phi.so``.  There is no CPU
fallback: if the library or a CUDA device is missing, every entry point
raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import ConfigError

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("MGP_LIB_PATH") or os.path.join(_PKG, "libmgrit_phi.so")
SRC_PATH = os.path.join(_PKG, "csrc", "mgrit_phi.cu")
HEADER_PATH = os.path.join(_ROOT, "include", "mgrit_phi.h")

MGP_OK, MGP_EINVAL, MGP_ECUDA = 0, 1, 2
SUM_SEQ, SUM_LANE2 = 0, 1
G_NONE, G_ZERO, G_ARRAY = 0, 1, 2
TAIL_NONE, TAIL_PHI, TAIL_RESTRICT, TAIL_RESID = 0, 1, 2, 3
SCHEME_RK_WENO, SCHEME_LF_ONESTEP, SCHEME_LF_MATCHED, SCHEME_RK_WENO_ROE = 0, 1, 2, 3
GUESS_LAST_STEP, GUESS_INJECTION = 0, 1
MODEL_BURGERS, MODEL_ADVECTION, MODEL_SHALLOW_WATER, MODEL_EULER = 0, 1, 2, 3
STATUS_NONPOSITIVE_DEPTH = 1
STATUS_NONPOSITIVE_DENSITY = 2
STATUS_NONPOSITIVE_PRESSURE = 4
STATUS_ROE_NONHYPERBOLIC = 8
ABI_VERSION = 6

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bit parity with NumPy: no FMA contraction, IEEE division and sqrt
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-diag-suppress", "128",
    "-Xcompiler", "-fPIC", "-shared",
]


class MgpPhi(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("weno_k", ctypes.c_int32),
                ("rk_order", ctypes.c_int32), ("regime", ctypes.c_int32),
                ("nx", ctypes.c_int64), ("dt", ctypes.c_double),
                ("dx", ctypes.c_double), ("epsilon", ctypes.c_double),
                ("speed", ctypes.c_double), ("scheme", ctypes.c_int32),
                ("lf_order", ctypes.c_int32), ("m_eff", ctypes.c_int32),
                ("repeats", ctypes.c_int32), ("gravity", ctypes.c_double),
                ("gamma", ctypes.c_double), ("characteristic", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


class MgpSweepArgs(ctypes.Structure):
    _fields_ = [
        ("phi", MgpPhi),
        ("n_chunks", _I64),
        ("start", _P), ("start_stride", _I64),
        ("n_steps", _I32), ("g_mode", _I32),
        ("g", _P), ("g_cs", _I64), ("g_ss", _I64),
        ("store", _P), ("st_cs", _I64), ("st_ss", _I64),
        ("tail", _I32), ("tail_regime", _I32),
        ("tail_g_mode", _I32), ("guess", _I32),
        ("tail_g", _P), ("tg_s", _I64),
        ("tail_out", _P), ("to_s", _I64),
        ("tail_out2", _P), ("to2_s", _I64),
        ("aux", _P), ("aux_s", _I64),
        ("aux2", _P), ("aux2_s", _I64),
        ("ref", _P), ("ref_cs", _I64), ("ref_ss", _I64),
        ("ref_last_next", _I32),
        ("count_nonfinite", _I32),
        ("partials", _P),
        ("status", _P),
    ]


class MgpFcfArgs(ctypes.Structure):
    _fields_ = [
        ("phi", MgpPhi),
        ("n_chunks", _I64),
        ("m", _I32), ("g_mode", _I32),
        ("cs", _P), ("cs_s", _I64),
        ("cd", _P), ("cd_s", _I64),
        ("fstore", _P), ("f_cs", _I64), ("f_ss", _I64),
        ("cstore", _P), ("cst_s", _I64),
        ("f0_start", _P),
        ("workspace", _P), ("workspace_bytes", _I64),
        ("epoch", ctypes.c_uint32), ("segment", _I32),
        ("split", _I32), ("reserved", _I32),
    ]


EXPORTED_SYMBOLS = ("mgp_sweep", "mgp_sum_partials", "mgp_max_nx",
                    "mgp_abi_version", "mgp_weno_tables", "mgp_launch_count",
                    "mgp_sweep_args_layout", "mgp_relax_fcf",
                    "mgp_relax_fcf_workspace")


N_PARTS = 7   # translation units of csrc/mgrit_phi.cu (MGP_PART, see the .cu)


def build(verbose: bool = False) -> str:
    """Compile libmgrit_phi.so for sm_100a with nvcc (no GPU needed): the
    source's N_PARTS kernel groups compile in parallel (-DMGP_PART=k, one
    process each), then one link.  MGP_BUILD_PARTS=0 compiles it as a single
    unit instead (same kernels, same flags)."""
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = ["-Xptxas=-v"] if verbose else []
    if os.environ.get("MGP_FAST_BUILD") == "1":
        # development builds: nvcc splits the optimiser over all host cores
        # (faster; the SASS schedule differs from the release build)
        extra.append("-split-compile=0")
    inc = ["-I", os.path.join(_ROOT, "include")]
    if os.environ.get("MGP_BUILD_PARTS", "1") == "0":
        subprocess.run([nvcc, *extra, *NVCC_FLAGS, *inc, "-o", LIB_PATH, SRC_PATH], check=True)
        return LIB_PATH
    obj_dir = os.path.join(_PKG, "build")
    os.makedirs(obj_dir, exist_ok=True)
    # each unit's fatbin compressed like the single-unit build's (nvcc leaves
    # smaller fatbins uncompressed by default)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + ["-Xfatbin=-compress-all"]
    objs, procs = [], []
    for k in range(1, N_PARTS + 1):
        obj = os.path.join(obj_dir, f"mgrit_phi.part{k}.o")
        objs.append(obj)
        procs.append(subprocess.Popen([nvcc, *extra, *compile_flags, *inc, f"-DMGP_PART={k}",
                                       "-c", "-o", obj, SRC_PATH]))
    bad = [k + 1 for k, pr in enumerate(procs) if pr.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, f"nvcc (MGP_PART {bad})")
    subprocess.run([nvcc, "-shared", "-Xcompiler", "-fPIC", "-o", LIB_PATH, *objs], check=True)
    return LIB_PATH


_lib = None


def load():
    """Load the library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.mgp_sweep.argtypes = [ctypes.POINTER(MgpSweepArgs), _P]
    lib.mgp_sweep.restype = ctypes.c_int
    lib.mgp_sum_partials.argtypes = [_P, _I64, _I32, _P, _P]
    lib.mgp_sum_partials.restype = ctypes.c_int
    lib.mgp_max_nx.argtypes = [_I32, _I32]
    lib.mgp_max_nx.restype = _I64
    lib.mgp_abi_version.restype = _I32
    dp = ctypes.POINTER(ctypes.c_double)
    lib.mgp_weno_tables.argtypes = [_I32, dp, dp, dp]
    lib.mgp_weno_tables.restype = ctypes.c_int
    lib.mgp_launch_count.restype = _I64
    lib.mgp_sweep_args_layout.argtypes = [ctypes.POINTER(_I64), _I32]
    lib.mgp_sweep_args_layout.restype = _I32
    lib.mgp_relax_fcf.argtypes = [ctypes.POINTER(MgpFcfArgs), _P]
    lib.mgp_relax_fcf.restype = ctypes.c_int
    lib.mgp_relax_fcf_workspace.argtypes = [ctypes.POINTER(MgpPhi), _I64, _I32]
    lib.mgp_relax_fcf_workspace.restype = _I64
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == MGP_OK:
        return
    if rc == MGP_EINVAL:
        raise ConfigError(f"{what}: invalid argument for the B200 kernels")
    raise RuntimeError(f"{what}: CUDA failure (status {rc})")


def launch_count() -> int:
    return int(load().mgp_launch_count())


def max_nx_static(weno_k: int = 2, model: int = 0) -> int:
    """The library's mesh limits (mgp_max_nx) without loading it: 4096 cells
    per CTA, WENO5 Burgers up to 16 x 4096 over a cluster, shallow water 2048."""
    if model in (MODEL_SHALLOW_WATER, MODEL_EULER):
        return 2048
    return 16 * 4096 if (weno_k == 2 and model == MODEL_BURGERS) else 4096


CTA_MAX_NX = 4096


def split_cluster_size(nx: int) -> int:
    """Cluster size the library splits a mesh of nx > 4096 cells over: the
    smallest cs in {2, 4, 8, 16} with nx % cs == 0 and nx / cs <= 4096, or 0
    if none exists (mgp_sweep then returns MGP_EINVAL) -- csrc split_cs."""
    for cs in (2, 4, 8, 16):
        if nx % cs == 0 and nx // cs <= CTA_MAX_NX:
            return cs
    return 0


def mesh_supported(nx: int, weno_k: int = 2, model: int = 0) -> bool:
    """nx within the kernel's limit and, above one CTA's 4096 cells, split
    evenly into power-of-two slabs (csrc validate())."""
    if nx > max_nx_static(weno_k, model):
        return False
    return nx <= CTA_MAX_NX or split_cluster_size(nx) > 0


def max_nx(weno_k: int = 2, model: int = 0) -> int:
    return int(load().mgp_max_nx(int(weno_k), int(model)))

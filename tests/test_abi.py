"""CPU: the C-ABI library loads and exports every symbol include/mgrit_phi.h
declares; the ctypes mirror of the argument structs matches the C layout;
the compile-time WENO tables equal float(Fraction) of weno.py:43-86.
No kernel is launched (there is no GPU here)."""
import ctypes
import re

import numpy as np
import pytest

from paper_2104_09404_b200 import _lib
from paper_2104_09404_b200.weno import build_tables


def _declared_functions():
    text = open(_lib.HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(mgp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_functions()
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name


def test_sweep_args_layout_matches_ctypes():
    lib = _lib.load()
    out = (ctypes.c_int64 * 64)()
    n = lib.mgp_sweep_args_layout(out, 64)
    fields = [f[0] for f in _lib.MgpSweepArgs._fields_]
    assert n == 2 + len(fields)
    assert out[0] == ctypes.sizeof(_lib.MgpPhi)
    assert out[1] == ctypes.sizeof(_lib.MgpSweepArgs)
    for i, name in enumerate(fields):
        assert out[2 + i] == getattr(_lib.MgpSweepArgs, name).offset, name


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_device_tables_equal_rational_tables(k):
    lib = _lib.load()
    cw = np.zeros(16)
    d = np.zeros(4)
    sm = np.zeros(64)
    dp = ctypes.POINTER(ctypes.c_double)
    assert lib.mgp_weno_tables(k, cw.ctypes.data_as(dp), d.ctypes.data_as(dp),
                               sm.ctypes.data_as(dp)) == 0
    t = build_tables(k)
    assert np.array_equal(cw.reshape(4, 4)[:k + 1, :k + 1], t.coeffs)
    assert np.array_equal(d[:k + 1], t.weights)
    assert np.array_equal(sm.reshape(4, 4, 4)[:k + 1, :k + 1, :k + 1], t.smoothness)


def test_abi_constants():
    lib = _lib.load()
    assert lib.mgp_abi_version() == _lib.ABI_VERSION
    assert lib.mgp_max_nx(2, 0) == 65536 and lib.mgp_max_nx(1, 0) == 4096
    assert lib.mgp_max_nx(2, 2) == 2048
    for k in range(4):
        for model in range(3):
            assert lib.mgp_max_nx(k, model) == _lib.max_nx_static(k, model)
    assert lib.mgp_launch_count() >= 0
    hdr = open(_lib.HEADER_PATH).read()
    for name, val in [("MGP_SUM_SEQ", _lib.SUM_SEQ), ("MGP_SUM_LANE2", _lib.SUM_LANE2),
                      ("MGP_G_ZERO", _lib.G_ZERO), ("MGP_G_ARRAY", _lib.G_ARRAY),
                      ("MGP_TAIL_PHI", _lib.TAIL_PHI), ("MGP_TAIL_RESTRICT", _lib.TAIL_RESTRICT),
                      ("MGP_TAIL_RESID", _lib.TAIL_RESID),
                      ("MGP_GUESS_INJECTION", _lib.GUESS_INJECTION),
                      ("MGP_MODEL_SHALLOW_WATER", _lib.MODEL_SHALLOW_WATER),
                      ("MGP_STATUS_NONPOSITIVE_DEPTH", _lib.STATUS_NONPOSITIVE_DEPTH),
                      ("MGP_SCHEME_RK_WENO_ROE", _lib.SCHEME_RK_WENO_ROE)]:
        assert re.search(rf"#define {name} {val}\b", hdr), name


def test_fcf_args_layout_matches_c_compiler(tmp_path):
    """The ctypes mirror of mgp_fcf_args against offsetof() from gcc on the
    header itself."""
    import subprocess
    fields = [f[0] for f in _lib.MgpFcfArgs._fields_]
    src = tmp_path / "layout.c"
    body = "".join(f'    printf("%zu\\n", offsetof(mgp_fcf_args, {f}));\n' for f in fields)
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "mgrit_phi.h"\n'
                   'int main(void) {\n    printf("%zu\\n", sizeof(mgp_fcf_args));\n'
                   + body + "    return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(_lib.os.path.dirname(_lib.HEADER_PATH)), "-o", str(exe),
                    str(src)], check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                           check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_lib.MgpFcfArgs)
    for name, off in zip(fields, vals[1:]):
        assert off == getattr(_lib.MgpFcfArgs, name).offset, name

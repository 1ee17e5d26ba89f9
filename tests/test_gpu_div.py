"""GPU: the shared-reciprocal division used for the WENO weights is
bit-identical to IEEE a / b (tests/cuda/div_check.cu)."""
import ctypes
import os

import pytest

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(__file__), "cuda", "libdivcheck.so")


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_div_shared_is_ieee_division(mode):
    lib = ctypes.CDLL(LIB)
    lib.div_check.restype = ctypes.c_int64
    lib.div_check.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_double)]
    w = (ctypes.c_double * 4)()
    for seed in (1, 2, 3, 4):
        bad = lib.div_check(seed * 7919 + mode, 1 << 24, mode, w)
        assert bad == 0, (mode, seed, bad, list(w))

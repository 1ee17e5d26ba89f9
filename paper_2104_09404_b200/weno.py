"""WENO reconstruction tables (host view).

The exact rational tables of reference ``pkg/src/mgritlab/weno.py:43-86``
re-derived here as Fractions and frozen to doubles; the device kernels carry
the same values as compile-time constants (``mgp_weno_tables`` exports them
so the tests can check both against these).  Reconstruction itself runs on
the GPU inside the fused propagator.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np

from .errors import ConfigError

DEFAULT_EPSILON = 1e-6
SUPPORTED_DEGREES = (0, 1, 2, 3)

_COEFFS = {
    0: (1, [[1]]),
    1: (2, [[1, 1], [-1, 3]]),
    2: (6, [[2, 5, -1], [-1, 5, 2], [2, -7, 11]]),
    3: (12, [[3, 13, -5, 1], [-1, 7, 7, -1], [1, -5, 13, 3], [-3, 13, -23, 25]]),
}
_WEIGHTS = {0: (1, [1]), 1: (3, [2, 1]), 2: (10, [3, 6, 1]), 3: (35, [4, 18, 12, 1])}
_SMOOTHNESS = {
    0: (1, [[[0]]]),
    1: (1, [[[1, -1], [-1, 1]], [[1, -1], [-1, 1]]]),
    2: (6, [[[20, -31, 11], [-31, 50, -19], [11, -19, 8]],
            [[8, -13, 5], [-13, 26, -13], [5, -13, 8]],
            [[8, -19, 11], [-19, 50, -31], [11, -31, 20]]]),
    3: (240, [[[2107, -4701, 3521, -927], [-4701, 11003, -8623, 2321],
               [3521, -8623, 7043, -1941], [-927, 2321, -1941, 547]],
              [[547, -1261, 961, -247], [-1261, 3443, -2983, 801],
               [961, -2983, 2843, -821], [-247, 801, -821, 267]],
              [[267, -821, 801, -247], [-821, 2843, -2983, 961],
               [801, -2983, 3443, -1261], [-247, 961, -1261, 547]],
              [[547, -1941, 2321, -927], [-1941, 7043, -8623, 3521],
               [2321, -8623, 11003, -4701], [-927, 3521, -4701, 2107]]]),
}


@dataclass(frozen=True)
class WenoTables:
    k: int
    coeffs: np.ndarray        # (k+1, k+1)
    weights: np.ndarray       # (k+1,)
    smoothness: np.ndarray    # (k+1, k+1, k+1)

    @property
    def order(self) -> int:
        return 2 * self.k + 1

    @property
    def window(self) -> int:
        return 2 * self.k + 1


@lru_cache(maxsize=None)
def build_tables(k: int) -> WenoTables:
    if k not in SUPPORTED_DEGREES:
        raise ConfigError(f"unsupported reconstruction degree k={k}, "
                          f"expected one of {SUPPORTED_DEGREES}")
    den, rows = _COEFFS[k]
    coeffs = np.array([[float(Fraction(v, den)) for v in row] for row in rows])
    den, vals = _WEIGHTS[k]
    weights = np.array([float(Fraction(v, den)) for v in vals])
    den, mats = _SMOOTHNESS[k]
    smooth = np.array([[[float(Fraction(v, den)) for v in row] for row in mat]
                       for mat in mats])
    return WenoTables(k=k, coeffs=coeffs, weights=weights, smoothness=smooth)

"""Canonical SHA-256 of a float64 array (test infrastructure): every NaN as
one bit pattern and -0.0 as +0.0 -- the only representation differences
between the GPU path and the oracle that DESIGN.md section 2 tolerates --
so full-size trajectories are compared bit for bit through a digest."""
import hashlib

import numpy as np


def canonical_hash(u) -> str:
    a = np.array(u, dtype=np.float64, copy=True).reshape(-1)
    a += 0.0                       # -0.0 + 0.0 = +0.0; other values unchanged
    a[np.isnan(a)] = np.nan        # one NaN bit pattern
    return hashlib.sha256(a.tobytes()).hexdigest()

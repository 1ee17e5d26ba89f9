"""CPU: the Euler / componentwise-system restatement in the oracle (test
infrastructure) against the reference (tests/golden/make_golden.py
"euler"): bit for bit against the reference run with its np.linalg.inv
replaced by the LU restatement (every other operation pinned), and within
1e-12 (max-norm relative, one step) of the unmodified reference, whose
LAPACK inverse differs in the last bits."""
import numpy as np
import pytest

import oracle


def params(c):
    return oracle.make_params(model=c["model"], k=c["k"], rk_order=c["rk"], dt=c["dt"],
                              dx=c["dx"], regime=oracle.SUM_LANE2,
                              scheme=3 if c["flux"] == "roe" else 0, gamma=c["gamma"],
                              gravity=c["gravity"], characteristic=c["characteristic"])


def close(a, b, tol=1e-12):
    fin = np.isfinite(b)
    if not np.array_equal(fin, np.isfinite(a)):
        return False
    if not fin.any():
        return True
    return np.max(np.abs(a[fin] - b[fin])) <= tol * np.max(np.abs(b[fin]))


def test_oracle_euler_vectors(euler_golden):
    index, data = euler_golden
    assert len(index) >= 170
    n_raise = n_exact_lapack = 0
    for c in index:
        u = data[c["key"] + "_in"]
        if c["raises"]:
            with pytest.raises(oracle.PhysicalStateOracleError):
                oracle.phi_apply(params(c), u, nthreads=1)
            n_raise += 1
            continue
        got = oracle.phi_apply(params(c), u, nthreads=1)
        assert np.array_equal(got, data[c["key"] + "_out_lu"], equal_nan=True), c
        assert close(got, data[c["key"] + "_out"]), c
        n_exact_lapack += np.array_equal(got, data[c["key"] + "_out"], equal_nan=True)
    assert n_raise >= 8
    # the LAPACK inverse only matters where eigenvectors are used
    assert n_exact_lapack > 0


def test_inverse_restatement_is_an_inverse():
    """inv3 (models.py:270 restated) on the Euler right-eigenvector matrices
    of random states: L @ R = I to rounding."""
    import json, os
    rng = np.random.default_rng(0)
    c = dict(model="euler", flux="lf", k=0, rk=0, dt=1e-3, dx=1 / 16, gamma=5 / 3,
             gravity=9.81, characteristic=True)
    u = np.empty((3, 16))
    u[0] = 1 + rng.random(16)
    u[1] = rng.standard_normal(16)
    u[2] = 3 + rng.random(16)
    # the rhs of a k=0 characteristic reconstruction equals the plain one
    # (L then R is the identity up to rounding)
    a = oracle.phi_apply(params(c), u, nthreads=1)
    b = oracle.phi_apply(params(dict(c, characteristic=False)), u, nthreads=1)
    assert close(a, b, 1e-12)

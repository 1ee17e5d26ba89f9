"""CPU: the shallow-water restatement in the oracle (test infrastructure) is
pinned to reference vectors (tests/golden/make_golden.py ``sw``): the
characteristic WENO reconstruction with LF and Roe fluxes (reference
flux.py:70-161, models.py:130-230) and the two checked-in shallow-water
configs (pkg/configs/high_order_shallow_water_{lf,roe}.cfg)."""
import numpy as np
import pytest

import oracle
from oracle import mgrit_oracle


def _params(c):
    return oracle.make_params(model="shallow-water", k=c["k"], rk_order=c["rk"],
                              dt=c["dt"], dx=c["dx"], regime=oracle.SUM_LANE2,
                              scheme=3 if c["flux"] == "roe" else 0, gravity=c["gravity"])


def test_oracle_matches_reference_sw_vectors(sw_golden):
    index, data = sw_golden
    assert len(index) >= 128
    raised = 0
    for c in index:
        u = data[c["key"] + "_in"]
        if c["raises"]:
            with pytest.raises(oracle.PhysicalStateOracleError):
                oracle.phi_apply(_params(c), u, nthreads=1)
            raised += 1
            continue
        got = oracle.phi_apply(_params(c), u, nthreads=1)
        assert np.array_equal(got, data[c["key"] + "_out"], equal_nan=True), c
    assert raised > 0


def _sw_steppers(spec):
    L, m = spec["n_levels"], spec["m"]
    orders = spec["weno_order"] * (L if len(spec["weno_order"]) == 1 else 1)
    rk = {"fe": 1, "ssprk2": 2, "ssprk3": 3}
    kinds = spec["stepper"] * (L if len(spec["stepper"]) == 1 else 1)
    dx = spec["length"] / spec["n_x"]
    return [oracle.OracleStepper(model="shallow-water", k=(orders[l] - 1) // 2,
                                 rk_order=rk[kinds[l]], dt=spec["dt"] * m ** l, dx=dx,
                                 scheme=3 if spec["flux"] == "roe" else 0,
                                 gravity=spec["gravity"], nthreads=1)
            for l in range(L)]


@pytest.mark.parametrize("name", ["high_order_shallow_water_lf__3",
                                  "high_order_shallow_water_roe__5"])
def test_oracle_sw_mgrit_matches_reference(sw_mgrit_golden, name):
    meta, data = sw_mgrit_golden
    spec = meta[name]
    st = _sw_steppers(spec)
    u0 = data[name + "__u0"]
    ref = mgrit_oracle.march(st[0], u0, spec["n_t"])
    opts = mgrit_oracle.Options(n_levels=spec["n_levels"], m=spec["m"], cycle=spec["cycle"],
                                relaxation=spec["relaxation"], guess=spec["guess"],
                                max_iters=spec["max_iters"])
    traj, rec = mgrit_oracle.mgrit_solve(st, u0, spec["n_t"], spec["dt"], opts, reference=ref)
    assert rec.diverged_at == spec["diverged_at"]
    np.testing.assert_allclose(rec.errors, data[name + "__errors"], rtol=1e-12, atol=0)
    assert np.array_equal(traj, data[name + "__traj"])

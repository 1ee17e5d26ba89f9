"""CPU: the oracle (test infrastructure) is pinned to golden vectors that
were produced by the reference itself (tests/golden/make_golden.py)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import mgrit_oracle


def _params(c, regime):
    return oracle.make_params(model=c["model"], k=c["k"], rk_order=c["rk"], dt=c["dt"],
                              dx=c["dx"], eps=c["eps"], speed=c["speed"], regime=regime)


def test_oracle_matches_reference_phi_vectors(phi_golden):
    index, data = phi_golden
    assert len(index) > 200
    for c in index:
        u = data[c["key"] + "_in"]
        want = data[c["key"] + "_out"]
        got = oracle.phi_apply(_params(c, oracle.regime_for_shape(u.shape)), u, nthreads=1)
        assert np.array_equal(got, want, equal_nan=True), c


def test_regime_matters_for_weno5(phi_golden):
    """The 2-lane / sequential candidate order is observable for k >= 2."""
    index, data = phi_golden
    flipped = 0
    for c in index:
        if c["k"] < 2 or c["field"] != "rough" or c["rk"] == 0:
            continue
        u = data[c["key"] + "_in"]
        want = data[c["key"] + "_out"]
        wrong = 1 - oracle.regime_for_shape(u.shape)
        got = oracle.phi_apply(_params(c, wrong), u, nthreads=1)
        flipped += not np.array_equal(got, want)
    assert flipped > 0


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_oracle_tables_are_rounded_fractions(k):
    from paper_2104_09404_b200.weno import build_tables
    cw, d, sm = oracle.tables(k)
    t = build_tables(k)
    assert np.array_equal(cw[:k + 1, :k + 1], t.coeffs)
    assert np.array_equal(d[:k + 1], t.weights)
    assert np.array_equal(sm[:k + 1, :k + 1, :k + 1], t.smoothness)
    # spot-check the Fraction rounding itself
    if k == 2:
        assert cw[2, 2] == float(Fraction(11, 6))
        assert sm[0, 0, 1] == float(Fraction(-31, 6))


def _oracle_run(spec, u0):
    L, m = spec["n_levels"], spec["m"]
    orders = spec["weno_order"] * (L if len(spec["weno_order"]) == 1 else 1)
    rk = {"fe": 1, "ssprk2": 2, "ssprk3": 3}
    kinds = spec["stepper"] * (L if len(spec["stepper"]) == 1 else 1)
    dx = spec.get("length", 1.0) / spec["n_x"]
    steppers = [oracle.OracleStepper(model=spec["model"], k=(orders[l] - 1) // 2,
                                     rk_order=rk[kinds[l]], dt=spec["dt"] * m ** l, dx=dx,
                                     speed=spec.get("speed", 1.0), nthreads=1)
                for l in range(L)]
    ref = None
    if spec["semantics"] == "harness":
        ref = mgrit_oracle.march(steppers[0], u0, spec["n_t"])
    opts = mgrit_oracle.Options(n_levels=L, m=m, cycle=spec["cycle"],
                                relaxation=spec["relaxation"], guess=spec["guess"],
                                max_iters=spec["max_iters"])
    return mgrit_oracle.mgrit_solve(steppers, u0, spec["n_t"], spec["dt"], opts, reference=ref)


FAST_CASES = ["c1_fcf_harness", "c2_scaled", "c2_scaled_converging", "c4_weno3_rk2_f",
              "fcycle_injection", "fcycle_fcf_laststep", "single_chunk",
              "high_order_burgers_lf_w5", "order_mix_space_time_down_lf"]


@pytest.mark.parametrize("name", FAST_CASES)
def test_oracle_mgrit_matches_reference_history(mgrit_golden, name):
    meta, data = mgrit_golden
    spec = meta[name]
    traj, rec = _oracle_run(spec, data[name + "__u0"])
    assert rec.diverged_at == spec["diverged_at"]
    want_r = data[name + "__residuals"]
    want_e = data[name + "__errors"]
    ok = np.isfinite(want_r)
    assert np.array_equal(np.isfinite(rec.residuals), ok)
    np.testing.assert_allclose(rec.residuals[ok], want_r[ok], rtol=1e-12, atol=0)
    oke = np.isfinite(want_e)
    np.testing.assert_allclose(rec.errors[oke], want_e[oke], rtol=1e-12, atol=0)
    if spec["has_traj"]:
        assert np.array_equal(traj, data[name + "__traj"], equal_nan=True)


def test_c1_known_answers(mgrit_golden):
    """SURVEY.md 8(d) C1 known answers (bit-sensitive): residual-only FCF
    row 1 = 7.67378330669847148e+90, row 63 = 1.53175844712423997e-02,
    row 64 = 0.0; F relaxation row 128 = 0.0."""
    _, data = mgrit_golden
    r = data["c1_fcf_residual_only__residuals"]
    assert r[1] == 7.67378330669847148e+90
    assert r[63] == 1.53175844712423997e-02
    assert r[64] == 0.0 and np.argmax(r < 1e-10) == 64
    rf = data["c1_f_residual_only__residuals"]
    assert rf[1] == 4.95406624397536612e+91
    assert rf[128] == 0.0 and np.argmax(rf < 1e-10) == 128

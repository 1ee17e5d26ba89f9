"""GPU parity of the one-step Lax-Friedrichs family (matched fine / coarse
order 0 and 1, rediscretised), of ComposedStepper and of the Roe flux with
entropy fix against the reference's own outputs -- propagator vectors and
the checked-in study configs (pkg/configs/fine_match_*, restriction_guess_*,
cfl_matched_fe, two_level_exact, fine_match_refinement_vcycle, *_roe)."""
import json
import os

import numpy as np
import pytest

import paper_2104_09404_b200 as P

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _stepper(c, sg):
    model = P.make_model("burgers")
    if c["kind"] == "roe":
        op = P.SemiDiscreteOperator(model, sg, P.FluxConfig("roe", P.WenoConfig(2 * c["k"] + 1)))
        return P.RungeKuttaStepper(op.rhs, c["dt"], c["rk"])
    if c["kind"] == "onestep":
        return P.MatchedLFFine(model, sg, c["dt"])
    if c["kind"] == "matched":
        return P.MatchedLFCoarse(model, sg, c["dt_fine"], c["m_eff"], c["order"])
    if c["inner"] == "fine":
        return P.ComposedStepper(P.MatchedLFFine(model, sg, c["dt_fine"]), c["repeats"])
    op = P.SemiDiscreteOperator(model, sg, P.FluxConfig("lf", P.WenoConfig(5)))
    return P.ComposedStepper(P.RungeKuttaStepper(op.rhs, c["dt_fine"], 3), c["repeats"])


def test_lf_vectors_match_reference():
    index = json.load(open(os.path.join(GOLDEN, "lf_vectors.json")))
    data = np.load(os.path.join(GOLDEN, "lf_vectors.npz"))
    for c in index:
        u = data[c["key"] + "_in"]
        sg = P.SpatialGrid(1.0, u.shape[-1])
        got = _stepper(c, sg).advance(u)
        assert np.array_equal(got, data[c["key"] + "_out"], equal_nan=True), c


def test_lf_study_configs_match_reference():
    meta = json.load(open(os.path.join(GOLDEN, "lf_mgrit_cases.json")))
    data = np.load(os.path.join(GOLDEN, "lf_mgrit_cases.npz"))
    for spec in meta:
        name = spec["name"]
        u0 = data[name + "__u0"]
        sg = P.SpatialGrid(spec["length"], spec["n_x"])
        tg = P.TemporalGrid(spec["horizon"], spec["n_t"])
        assert tg.dt == spec["dt"]
        steppers = P.build_steppers(P.make_model("burgers"), sg, tg, n_levels=spec["n_levels"],
                                    m=spec["m"], weno_order=spec["weno_order"],
                                    stepper=spec["stepper"], coarse=spec["coarse"],
                                    flux=spec.get("flux", "lf"))
        serial = P.solve_serial(steppers[0], u0, tg, sg, P.make_model("burgers"))
        opts = P.MgritOptions(n_levels=spec["n_levels"], m=spec["m"], cycle=spec["cycle"],
                              relaxation=spec["relaxation"], guess=spec["guess"],
                              max_iters=spec["max_iters"])
        _, rec = P.mgrit_solve(steppers, u0, tg, sg, opts, reference=serial.device_values,
                               return_trajectory=False)
        assert rec.diverged_at == spec["diverged_at"], name
        for what in ("errors", "residuals"):
            want = data[f"{name}__{what}"]
            got = getattr(rec, what)
            ok = np.isfinite(want)
            assert np.array_equal(np.isfinite(got), ok), (name, what)
            np.testing.assert_allclose(got[ok], want[ok], rtol=1e-10, atol=0, err_msg=name)
            assert np.array_equal(got[ok] == 0.0, want[ok] == 0.0), (name, what)

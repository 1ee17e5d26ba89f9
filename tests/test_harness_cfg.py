"""CPU: the experiment harness (reference harness.py:88-495) -- config
parsing and validation, sweeps, CSV / meta formats -- and, through the
mgp_sweep emulator, one checked-in config end to end against the table the
reference wrote (tests/golden/config_tables.json)."""
import json
import os

import numpy as np
import pytest

import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import harness as H

import sweep_emulator

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

TEXT = """# a comment line
problem = burgers
ic = burgers-43     # trailing comment
L = 2.0
T = 0.5
N_x = 64
N_t = 400
n_levels = 3
stepper = ssprk3/ssprk2/fe
weno_order = 5/3/1
characteristic = off
sweep = N_x
sweep_values = 32, 64
"""


def test_parse_config_keys_aliases_sweeps():
    c = P.parse_config(TEXT)
    assert (c.problem, c.ic, c.length, c.horizon, c.n_x, c.n_t) == \
        ("burgers", "burgers-43", 2.0, 0.5, 64, 400)
    assert c.stepper == ("ssprk3", "ssprk2", "fe") and c.weno_order == (5, 3, 1)
    assert c.characteristic is False
    assert c.sweep == "n_x" and c.sweep_values == ("32", "64")
    assert c.m == 2 and c.cycle == "v" and c.relaxation == "f" and c.max_iters == 10
    col = P.apply_sweep_value(c, c.sweep, "32")
    assert col.n_x == 32
    grid = P.apply_sweep_value(c, "grid", "128x800")
    assert (grid.n_x, grid.n_t) == (128, 800)
    with pytest.raises(P.ConfigError):
        P.apply_sweep_value(c, "grid", "128by800")


@pytest.mark.parametrize("text,line,key", [
    ("problem burgers", 1, None),
    ("problem = burgers\nfoo = 1", 2, "foo"),
    ("problem = burgers\nproblem = burgers", 2, "problem"),
    ("problem =", 1, "problem"),
    ("problem = burgers\nic = sin-moving\nT = 1\nN_x = x2\nN_t = 4\nn_levels = 2", 4, "n_x"),
    ("problem = burgers\nic = sin-moving\nT = 1\nN_x = 8\nN_t = 4", None, "n_levels"),
    ("problem = burgers\nic = sin-moving\nT = 1\nN_x = 8\nN_t = 4\nn_levels = 2\nsweep = m",
     None, "sweep"),
])
def test_parse_errors_name_line_and_key(text, line, key):
    with pytest.raises(P.ParseError) as e:
        P.parse_config(text)
    assert e.value.line == line and e.value.key == key


BASE = "problem = {p}\nic = {ic}\nT = 1\nN_x = 16\nN_t = 8\nn_levels = 2\n"


@pytest.mark.parametrize("extra,p,ic", [
    ("", "burgers", "sw-scaled"),                       # ic of another model
    ("m = 3\n", "burgers", "sin-moving"),               # N_t not divisible
    ("stepper = matched-lf\n", "shallow-water", "sw-scaled"),
    ("coarse = matched-1\n", "burgers", "sin-moving"),  # needs matched-lf
    ("stepper = fe/fe/fe\n", "burgers", "sin-moving"),  # wrong per-level count
    ("coarse = exact\nweno_order = 1/3\n", "burgers", "sin-moving"),
    ("flux = hll\n", "burgers", "sin-moving"),
    ("cycle = w\n", "burgers", "sin-moving"),
])
def test_validate_rejections(extra, p, ic):
    with pytest.raises(P.ConfigError):
        P.parse_config(BASE.format(p=p, ic=ic) + extra)


def test_csv_and_meta_formats(tmp_path):
    t = P.ConvergenceTable(columns=["a=1", "b"],
                           data=np.array([[0.1, np.nan], [1e-300, 2.5]]))
    out = tmp_path / "x.csv"
    P.emit_csv(t, out)
    assert out.read_bytes() == b"iteration,a=1,b\n0,0.1,NaN\n1,1e-300,2.5\n"
    rec = P.ConvergenceRecord(errors=np.array([1.0, np.nan]), residuals=np.zeros(2),
                              diverged=True, diverged_at=1)
    cfg = P.ExperimentConfig(problem="burgers", ic="sin-moving", horizon=1.0, n_x=16,
                             n_t=8, n_levels=2)

    class S:
        wall_seconds = 0.25

    res = P.ExperimentResult(config=cfg, record=rec, serial=S(), level_dts=(0.125, 0.25),
                             level_cfls=(0.1234567, 0.2469134), wall_seconds=1.5)
    P.write_meta(out, ["col"], [res])
    assert P.meta_path(out).read_text() == (
        "[col]\nproblem = burgers\nic = sin-moving\nn_x = 16\nn_t = 8\nn_levels = 2\n"
        "level_dt = 0.125, 0.25\nlevel_cfl = 0.123457, 0.246913\n"
        "serial_wall_seconds = 0.250\nwall_seconds = 1.500\ndiverged = true\n"
        "diverged_at = 1\n\ntotal_wall_seconds = 1.500\n")


def _golden():
    return {g["name"]: g for g in json.load(open(os.path.join(GOLDEN, "config_tables.json")))}


def config_of(g):
    f = dict(g["config"])
    for k in ("weno_order", "stepper", "sweep_values"):
        f[k] = tuple(f[k])
    return P.ExperimentConfig(**f)


def read_csv(text):
    lines = text.rstrip("\n").split("\n")
    header = lines[0].split(",")
    rows = np.array([[float(v) for v in ln.split(",")[1:]] for ln in lines[1:]])
    return header, rows


def test_golden_configs_validate():
    gold = _golden()
    assert len(gold) == 22
    for g in gold.values():
        P.validate_config(config_of(g))


def test_config_end_to_end_emulated(tmp_path):
    """two_level_exact.cfg (matched-lf fine, exact composed coarse) through
    run_experiment / emit_csv with emulated kernels."""
    g = _golden()["two_level_exact"]
    sweep_emulator.install()
    try:
        res = P.run_experiment(config_of(g))
    finally:
        sweep_emulator.remove()
    out = tmp_path / "t.csv"
    P.emit_csv(P.experiment_table(res), out)
    h1, r1 = read_csv(out.read_text())
    h0, r0 = read_csv(g["csv"])
    assert h1 == h0 and r1.shape == r0.shape
    np.testing.assert_allclose(r1, r0, rtol=1e-10, atol=0, equal_nan=True)
    np.testing.assert_allclose(res.level_cfls, g["level_cfls"][0], rtol=1e-14)

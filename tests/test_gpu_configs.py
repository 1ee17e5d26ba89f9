"""GPU: every checked-in reference config (pkg/configs/*.cfg except the two
Euler ones, outside the path) through run_sweep / run_experiment ->
emit_csv, against the CSV the reference harness wrote for it
(tests/golden/config_tables.json): same columns and rows, NaN exactly where
the reference diverged, errors within the north-star 1e-10 relative,
per-level CFL numbers equal, and the GPU table deterministic byte for byte."""
import json
import os

import numpy as np
import pytest

import paper_2104_09404_b200 as P

from test_harness_cfg import config_of, read_csv

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GOLD = json.load(open(os.path.join(GOLDEN, "config_tables.json")))


def _run(cfg):
    if cfg.sweep is not None:
        res = P.run_sweep(cfg)
        return res.table, res.runs
    run = P.run_experiment(cfg)
    return P.experiment_table(run), [run]


@pytest.mark.parametrize("g", GOLD, ids=[g["name"] for g in GOLD])
def test_config_table_matches_reference(g, tmp_path):
    table, runs = _run(config_of(g))
    out = tmp_path / "t.csv"
    P.emit_csv(table, out)
    h1, r1 = read_csv(out.read_text())
    h0, r0 = read_csv(g["csv"])
    assert h1 == h0
    assert r1.shape == r0.shape
    assert np.array_equal(np.isnan(r1), np.isnan(r0))
    np.testing.assert_allclose(r1, r0, rtol=1e-10, atol=0, equal_nan=True)
    for run, dts, cfls, vmax, dv in zip(runs, g["level_dts"], g["level_cfls"],
                                        g["max_speed"], g["diverged_at"]):
        assert list(run.level_dts) == dts
        assert run.serial.max_speed == vmax
        np.testing.assert_allclose(run.level_cfls, cfls, rtol=1e-15)
        assert run.record.diverged_at == dv
    P.write_meta(out, table.columns, runs)
    assert P.meta_path(out).read_text().count("level_cfl = ") == len(runs)


def test_config_csv_is_deterministic(tmp_path):
    g = next(x for x in GOLD if x["name"] == "high_order_shallow_water_roe")
    payloads = []
    for i in range(2):
        table, _ = _run(config_of(g))
        out = tmp_path / f"t{i}.csv"
        P.emit_csv(table, out)
        payloads.append(out.read_bytes())
    assert payloads[0] == payloads[1]

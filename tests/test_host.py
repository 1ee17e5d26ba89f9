"""CPU: host-side API mirror -- validation and error conventions follow the
reference (ConfigError at construction), problem set-up, no CPU fallback."""
import numpy as np
import pytest

import paper_2104_09404_b200 as P
from paper_2104_09404_b200 import harness


def test_config_errors_mirror_reference():
    with pytest.raises(P.ConfigError):
        P.WenoConfig(order=4)
    with pytest.raises(P.ConfigError):
        P.WenoConfig(order=5, epsilon=0.0)
    with pytest.raises(P.ConfigError):
        P.FluxConfig(kind="hll")
    sg = P.SpatialGrid(1.0, 4)
    with pytest.raises(P.ConfigError):   # 4 cells cannot support WENO5 (flux.py:138-141)
        P.SemiDiscreteOperator(P.make_model("burgers"), sg, P.FluxConfig("lf", P.WenoConfig(5)))
    with pytest.raises(P.ConfigError):   # Roe: Burgers and the systems, not advection
        P.SemiDiscreteOperator(P.make_model("advection"), P.SpatialGrid(1.0, 8),
                               P.FluxConfig("roe", P.WenoConfig(1)))
    with pytest.raises(P.ConfigError):   # matched operators: scalar Burgers only
        P.MatchedLFFine(P.make_model("advection"), P.SpatialGrid(1.0, 8), 0.1)
    with pytest.raises(P.ConfigError):
        P.MatchedLFCoarse(P.make_model("burgers"), P.SpatialGrid(1.0, 8), 0.1, 2, 2)
    with pytest.raises(P.ConfigError):
        P.make_model("navier-stokes")
    with pytest.raises(P.PhysicalStateError):    # models.py:219-223
        P.make_model("euler", gamma=1.0)
    with pytest.raises(P.ConfigError):           # beyond the system kernel's mesh limit
        P.SemiDiscreteOperator(P.make_model("euler"), P.SpatialGrid(1.0, 4096),
                               P.FluxConfig("roe", P.WenoConfig(3)))
    # WENO5 Burgers above 4096 cells: only meshes that split into 2/4/8/16
    # equal slabs of <= 4096 cells (the library returns MGP_EINVAL otherwise)
    for bad_nx in (8193, 8202, 9003, 65535):
        assert not P._lib.mesh_supported(bad_nx)
        with pytest.raises(P.ConfigError):
            P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, bad_nx),
                                   P.FluxConfig("lf", P.WenoConfig(5)))
    for good_nx, cs in ((8190, 2), (8192, 2), (12288, 4), (65536, 16), (40000, 16)):
        assert P._lib.split_cluster_size(good_nx) == cs, good_nx
        P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, good_nx),
                               P.FluxConfig("lf", P.WenoConfig(5)))
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, 8),
                                P.FluxConfig("lf", P.WenoConfig(3)))
    with pytest.raises(P.ConfigError):
        P.RungeKuttaStepper(op.rhs, 0.1, 4)
    with pytest.raises(P.ConfigError):
        P.RungeKuttaStepper(op.rhs, -0.1, 3)
    with pytest.raises(P.ConfigError):
        P.RungeKuttaStepper(lambda u: u, 0.1, 3)
    for bad in (dict(n_levels=1), dict(n_levels=2, m=1), dict(n_levels=2, cycle="w"),
                dict(n_levels=2, relaxation="cf"), dict(n_levels=2, guess="zero"),
                dict(n_levels=2, max_iters=-1), dict(n_levels=2, parallelism=0)):
        with pytest.raises(P.ConfigError):
            P.MgritOptions(**bad)


def test_hierarchy_checks_before_touching_the_device():
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, 8),
                                P.FluxConfig("lf", P.WenoConfig(3)))
    st = P.RungeKuttaStepper(op.rhs, 0.01, 3)
    u0 = np.zeros((1, 8))
    with pytest.raises(P.ConfigError):
        P.MgritHierarchy([st], u0, P.TemporalGrid(1.0, 8), P.SpatialGrid(1.0, 8),
                         P.MgritOptions(n_levels=2))
    with pytest.raises(P.ConfigError):   # 10 not divisible by m^(L-1) = 4
        P.MgritHierarchy([st, st, st], u0, P.TemporalGrid(1.0, 10),
                         P.SpatialGrid(1.0, 8), P.MgritOptions(n_levels=3, m=2))


def test_baseline_configs():
    c = P.BASELINE_CONFIGS
    assert P.auto_levels(65536, 4) == 7 == c["c3"].n_levels
    assert P.auto_levels(262144, 16) == 5 == c["c5"].n_levels
    assert c["c1"].time_grid().dt == 0.5 / 128
    assert len(P.c4_grid()) == 192
    u0 = c["c2"].initial_state()
    assert u0.shape == (1, 512)
    tg = c["c2"].time_grid(u0)
    assert abs(tg.dt - 0.4 * (1 / 512) / np.max(np.abs(u0))) < 1e-18
    # seeded IC is reproducible and draws all a before all phi
    a, phi = harness.fourier_modes(4, 1234)
    rng = np.random.default_rng(1234)
    assert np.array_equal(a, rng.uniform(-0.25, 0.25, 4))
    assert np.array_equal(phi, rng.uniform(0, 2 * np.pi, 4))
    counts = c["c3"].relaxation_phi_per_iteration()
    assert counts["relaxation"] == 218400 and counts["restriction"] == 43680
    assert c["c2"].relaxation_phi_per_iteration()["relaxation"] == 10240


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    op = P.SemiDiscreteOperator(P.make_model("burgers"), P.SpatialGrid(1.0, 8),
                                P.FluxConfig("lf", P.WenoConfig(3)))
    st = P.RungeKuttaStepper(op.rhs, 0.01, 3)
    with pytest.raises(RuntimeError):
        st.advance(np.zeros((2, 1, 8)))

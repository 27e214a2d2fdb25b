"""Host-side API semantics (no GPU): meshes, time plans, moments, boundary
specs, collision models and config packing -- mirroring the reference's
test_mesh.py / test_gas_state.py / test_boundary.py expectations."""

import math

import numpy as np
import pytest

from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, ConfigurationError,
                                   EXTRAPOLATE, InvalidStateError, PERIODIC, PhaseMesh,
                                   WallSpec, cell_centers, conserved_2d, plan_time,
                                   primitives_2d)


def test_axis_centres_and_spacing():
    ax = Axis(-8.0, 8.0, 64)
    c = cell_centers(ax)
    assert ax.spacing == 0.25
    assert c[0] == -7.875 and c[-1] == 7.875
    assert ax.center(1) == c[0]
    assert ax.vmax_abs == 8.0
    with pytest.raises(ConfigurationError):
        Axis(1.0, 0.0, 4)
    with pytest.raises(ConfigurationError):
        Axis(0.0, 1.0, 0)


def test_plan_time_lands_on_t_final():
    mesh = PhaseMesh(space=(Axis(0, 1, 512), Axis(0, 1, 512)),
                     velocity=(Axis(-8, 8, 32), Axis(-8, 8, 32)))
    plan = plan_time(0.1, 0.4, mesh)
    assert plan.n_steps == 1024
    assert plan.dt == pytest.approx(9.765625e-5, rel=1e-15)
    assert plan.n_steps * plan.dt == pytest.approx(0.1, rel=1e-14)
    assert plan.cfl_effective <= 0.4 + 1e-15
    with pytest.raises(ConfigurationError):
        plan_time(0.1, 1.2, mesh)


def test_conserved_primitive_round_trip():
    rng = np.random.default_rng(0)
    rho = rng.uniform(0.5, 2, (5, 4))
    u1, u2 = rng.uniform(-1, 1, (2, 5, 4))
    t11, t22 = rng.uniform(0.5, 1.5, (2, 5, 4))
    t12 = 0.1 * rng.uniform(-1, 1, (5, 4))
    Q = conserved_2d(rho, u1, u2, t11, t12, t22)
    r, a, b, tt, T, p = primitives_2d(Q)
    np.testing.assert_allclose(r, rho, rtol=1e-15)
    np.testing.assert_allclose(tt.t12, t12, atol=1e-14)
    np.testing.assert_allclose(T, 0.5 * (t11 + t22), rtol=1e-13)


def test_invalid_state_names_first_cell():
    Q = conserved_2d(np.ones((4, 3)), 0.0, 0.0, 1.0, 0.0, 1.0)
    Q[2, 1, 0] = -1.0
    Q[3, 0, 0] = -2.0
    with pytest.raises(InvalidStateError) as ei:
        primitives_2d(Q)
    assert ei.value.cell == (2, 1)
    assert ei.value.value == -1.0


def test_boundary_spec_validation():
    BoundarySpec2D(PERIODIC, PERIODIC, EXTRAPOLATE, WallSpec(1.0, 0.2))
    with pytest.raises(ConfigurationError):
        BoundarySpec2D(PERIODIC, EXTRAPOLATE, PERIODIC, PERIODIC)
    with pytest.raises(ConfigurationError):
        WallSpec(0.0)
    with pytest.raises(ConfigurationError):
        BoundarySpec2D("outflow", EXTRAPOLATE, PERIODIC, PERIODIC)


def test_collision_models():
    m = CollisionModel("esbgk_2d", nu=-0.5)
    assert m.tau(2.0, 1.0) == pytest.approx(2 * 0.4625 * math.pi)
    assert CollisionModel("bgk_2d").tau(1.0, 1.0) == pytest.approx(3 * math.pi * 0.436 / math.sqrt(2))
    assert CollisionModel("constant", value=0.7).tau(np.ones(3), 1.0).tolist() == [0.7] * 3
    with pytest.raises(ConfigurationError):
        CollisionModel("esbgk_2d", nu=1.0)
    with pytest.raises(ConfigurationError):
        CollisionModel("nope")


def test_config_packing_matches_problem():
    from paper_2509_21832_b200.solver import make_config
    mesh = PhaseMesh(space=(Axis(0, 1, 16), Axis(0, 2, 8)),
                     velocity=(Axis(-7, 7, 32), Axis(-6, 6, 30)))
    bc = BoundarySpec2D(WallSpec(1.0), WallSpec(1.1), EXTRAPOLATE, WallSpec(1.0, 0.16))
    cfg = make_config(mesh, bc, 0.05, CollisionModel("esbgk_2d", nu=-0.5), grid=(2, 1),
                      rank=(1, 0))
    assert (cfg.nx, cfg.ny, cfg.nv1, cfg.nv2) == (16, 8, 32, 30)
    assert list(cfg.face) == [2, 2, 1, 2]
    assert cfg.wall_T[1] == 1.1 and cfg.wall_U[3] == 0.16
    assert (cfg.px, cfg.py, cfg.rx, cfg.ry) == (2, 1, 1, 0)
    assert cfg.tau_kind == 2 and cfg.nu == -0.5 and cfg.eps == 0.05


def test_device_path_fails_loudly_without_gpu():
    """No CPU fallback: asking for the device path without CUDA raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_21832_b200 import NativeLibraryError, step_2d
    mesh = PhaseMesh(space=(Axis(0, 1, 4), Axis(0, 1, 4)),
                     velocity=(Axis(-5, 5, 4), Axis(-5, 5, 4)))
    bc = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
    from paper_2509_21832_b200 import State2D
    st = State2D(0.0, conserved_2d(np.ones((4, 4)), 0, 0, 1, 0, 1), np.zeros((4, 4, 4, 4)))
    with pytest.raises(NativeLibraryError):
        step_2d(st, mesh, bc, 0.1, CollisionModel("esbgk_2d"), 1e-3)


def test_run_driver_host_helpers():
    """snap-step mapping, steady window and totals follow cases.py:178-222."""
    from paper_2509_21832_b200.runner.drive import snap_steps, steady_window, totals
    # nearest step, clipped to [1, n], first request wins; Python round (half to even)
    assert snap_steps([0.01, 0.011, 0.5, 2.0, 0.0], 0.004, 100) == {2: 0.01, 3: 0.011, 100: 0.5, 1: 0.0}
    assert snap_steps([0.01, 0.0101], 0.004, 100) == {2: 0.01, 3: 0.0101}
    assert steady_window(7) == 1 and steady_window(100) == 10 and steady_window(101) == 11
    Q = np.arange(2 * 3 * 6, dtype=float).reshape(2, 3, 6)
    assert totals(Q, 0.5) == tuple(float(v) for v in Q.reshape(-1, 6).sum(axis=0) * 0.5)


def test_heat_flux_vector_matches_reference_formula():
    from paper_2509_21832_b200.macro2d import heat_flux_vector_2d
    rng = np.random.default_rng(3)
    h = rng.normal(size=(4, 5, 6))
    hx, hy = heat_flux_vector_2d(*h)
    assert np.array_equal(hx, 0.5 * (h[0] + h[2])) and np.array_equal(hy, 0.5 * (h[1] + h[3]))

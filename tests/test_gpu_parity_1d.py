"""GPU parity of the 1D1V path (BASELINE config 1) through the public API and
the C ABI (include/mm1d.h): the generic two-kernel step and the
cluster-resident run kernel, against the reference goldens, the CPU oracle
and the reference's frozen mms_run_1d(10) pin.

Tolerances as for 2D: moments 1e-11 relative after one step, 1e-9 after
many; the micro field 1e-10 of its maximum.
"""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, problem1d_from_golden, q1_rel_err, rel_err

pytestmark = pytest.mark.gpu

TOL_1, TOL_N, TOL_G = 1e-11, 1e-9, 1e-10


@pytest.fixture(scope="module")
def mm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200 import _native
    _native.load()
    return mm


@pytest.mark.parametrize("name", golden_cases("step1d_"))
def test_step1d_matches_reference_goldens(mm, name):
    mesh, bc, eps, model, p = problem1d_from_golden(name)
    d = np.load(GOLDEN / f"{name}.npz")
    st = mm.State1D(0.0, d["Q0"], d["G0"])
    dt = float(d["dt"])
    for n in range(1, max(p["steps"]) + 1):
        st = mm.step_1d(st, mesh, bc, eps, model, dt)
        if n in p["steps"]:
            assert q1_rel_err(st.Q, d[f"Q{n}"]) <= (TOL_1 if n == 1 else TOL_N), n
            assert rel_err(st.G, d[f"G{n}"]) <= TOL_G, n


@pytest.mark.parametrize("name", golden_cases("step1d_"))
@pytest.mark.parametrize("resident", [True, False])
def test_run1d_matches_oracle(mm, oracle, name, resident, monkeypatch):
    """run path (cluster-resident kernel, or the graph replay when disabled)
    for 150 steps against the oracle, including H of the last step."""
    from paper_2509_21832_b200.solver1d import Solver1D
    if not resident:
        monkeypatch.setenv("MM1D_NO_RESIDENT", "1")
    mesh, bc, eps, model, p = problem1d_from_golden(name)
    d = np.load(GOLDEN / f"{name}.npz")
    s = Solver1D(mesh, bc, eps, model)
    assert s.resident == resident
    dt, n = float(d["dt"]), 150
    Q, G, H = s.run_host(d["Q0"], d["G0"], dt, n)
    prob = oracle.Problem1D(mesh, bc, eps, model)
    Qo, Go = d["Q0"], d["G0"]
    for _ in range(n):
        Qo, Go, Ho = oracle.step_1d_arrays(prob, Qo, Go, dt)
    assert q1_rel_err(Q, Qo) <= TOL_N
    assert rel_err(G, Go) <= TOL_G
    assert rel_err(H, Ho) <= TOL_G
    s.close()


def sod_config1(mm):
    """BASELINE configs[0]: Sod tube, Nx=256, 64 velocities on [-8, 8], eps=1e-2,
    outflow (EXTRAPOLATE) faces, hard_sphere_1d tau, CFL 0.4 to t=0.1."""
    from paper_2509_21832_b200 import (EXTRAPOLATE, Axis, BoundarySpec1D, CollisionModel,
                                       PhaseMesh, cell_centers)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, 256),), velocity=(Axis(-8.0, 8.0, 64),))
    bc = BoundarySpec1D(EXTRAPOLATE, EXTRAPOLATE)
    x = cell_centers(mesh.space[0])
    left = x < 0.5
    rho = np.where(left, 1.0, 0.125)
    T = np.where(left, 1.0, 0.8)
    return mesh, bc, 1e-2, CollisionModel("hard_sphere_1d"), rho, np.zeros_like(rho), T


def test_config1_full_run_matches_oracle(mm, oracle):
    """The whole config-1 run (512 steps) in one resident launch vs the oracle."""
    mesh, bc, eps, model, rho, u, T = sod_config1(mm)
    G0 = np.zeros((256, 64))
    st, plan = mm.run_1d(mesh, bc, eps, model, rho, u, T, G0, 0.1, 0.4)
    assert plan.n_steps == 512
    prob = oracle.Problem1D(mesh, bc, eps, model)
    Q, G = mm.conserved_1d(rho, u, T), G0
    for _ in range(plan.n_steps):
        Q, G, _ = oracle.step_1d_arrays(prob, Q, G, plan.dt)
    assert q1_rel_err(st.Q, Q) <= TOL_N
    assert rel_err(st.G, G) <= TOL_G
    # conservation of mass up to the outflow fluxes is not exact; positivity is
    assert np.all(st.Q[:, 0] > 0)


def test_mms1d_regression_pin_on_gpu(mm):
    """mms_run_1d(10) through step_1d with the MMS source hooks: the
    reference's frozen errors (test_cases.py:98-102) at rel 1e-12."""
    from test_oracle_golden import mms1d_problem, relative_l2
    mesh, bc, eps, model, exact, msrc, qsrc = mms1d_problem(10)
    plan = mm.plan_time(0.9351, 0.95, mesh)
    Q0, G0 = exact(0.0)
    st = mm.State1D(0.0, Q0, G0)
    for n in range(plan.n_steps):
        st = mm.step_1d(st, mesh, bc, eps, model, plan.dt, micro_source=msrc,
                        macro_source=qsrc)
        st.t = (n + 1) * plan.dt
    Qe, Ge = exact(0.9351)
    assert relative_l2(st.Q, Qe) == pytest.approx(0.06653393519741775, rel=1e-12)
    assert relative_l2(st.G, Ge) == pytest.approx(0.09812773373649085, rel=1e-12)


def _bad_state(kind):
    from paper_2509_21832_b200 import (EXTRAPOLATE, Axis, BoundarySpec1D, CollisionModel,
                                       PhaseMesh)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, 16),), velocity=(Axis(-6.0, 6.0, 24),))
    bc = BoundarySpec1D(EXTRAPOLATE, EXTRAPOLATE)
    Q = np.tile([1.0, 0.1, 1.0], (16, 1))
    if kind == "density":
        Q[5, 0] = -0.25
        Q[9, 0] = -1.0
        want = ((5,), -0.25, "non-positive density")
    else:
        Q[7, 2] = 0.001     # T = 2E/rho - u^2 < 0
        want = ((7,), 2 * 0.001 - 0.01, "non-positive temperature")
    return mesh, bc, 0.05, CollisionModel("hard_sphere_1d"), Q, np.zeros((16, 24)), want


@pytest.mark.parametrize("kind", ["density", "temperature"])
def test_step1d_raises_reference_error(mm, kind):
    mesh, bc, eps, model, Q, G, (cell, value, msg) = _bad_state(kind)
    st = mm.step_1d(mm.State1D(0.0, Q, G), mesh, bc, eps, model, 1e-3)
    with pytest.raises(mm.InvalidStateError) as ei:
        st.Q
    assert tuple(ei.value.cell) == cell
    assert ei.value.value == pytest.approx(value, rel=1e-14)
    assert msg in str(ei.value)
    # the reference raises the same error
    with pytest.raises(mm.InvalidStateError) as ref:
        mm.primitives_1d(Q)
    assert tuple(ref.value.cell) == cell


@pytest.mark.parametrize("kind", ["density", "temperature"])
def test_run1d_resident_raises_reference_error(mm, kind):
    from paper_2509_21832_b200.solver1d import Solver1D
    mesh, bc, eps, model, Q, G, (cell, value, msg) = _bad_state(kind)
    s = Solver1D(mesh, bc, eps, model)
    assert s.resident
    with pytest.raises(mm.InvalidStateError) as ei:
        s.run_host(Q, G, 1e-3, 20)
    assert tuple(ei.value.cell) == cell
    assert ei.value.value == pytest.approx(value, rel=1e-14)
    # the context is usable again after the error was reported
    Qg = np.tile([1.0, 0.1, 1.0], (16, 1))
    Qr, _, _ = s.run_host(Qg, G, 1e-3, 3)
    assert np.all(np.isfinite(Qr))
    s.close()


def test_resident_and_step_paths_agree(mm):
    """Same 40 steps through step_1d (two kernels per step) and through one
    resident launch: identical up to reduction order."""
    from paper_2509_21832_b200.solver1d import Solver1D
    mesh, bc, eps, model, rho, u, T = sod_config1(mm)
    Q0 = mm.conserved_1d(rho, u, T)
    G0 = np.zeros((256, 64))
    dt = 1.953125e-4
    s = Solver1D(mesh, bc, eps, model)
    Qr, Gr, _ = s.run_host(Q0, G0, dt, 40)
    st = mm.State1D(0.0, Q0, G0)
    for _ in range(40):
        st = mm.step_1d(st, mesh, bc, eps, model, dt)
    assert q1_rel_err(Qr, st.Q) <= 1e-12
    assert rel_err(Gr, st.G) <= 1e-11
    s.close()

"""The device run driver (runner/drive.py: the reference's ``_advance``,
cases.py:199-231) against the same loop driven by the CPU oracle: final
state, frames at the requested times (``frame_2d`` moments, H about
u^{n+1}), the steady-state change over the last 10% of steps, the step
cap, and the MMS-source path."""

import numpy as np
import pytest

from conftest import GOLDEN, problem_from_golden, q_rel_err, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2509_21832_b200 as mm
    return mm


def oracle_advance(oracle, mesh, bc, eps, model, Q, G, t_final, cfl, frame_times, max_steps,
                   track_steady):
    """_advance restated on the oracle (cases.py:199-231)."""
    from paper_2509_21832_b200 import plan_time
    from paper_2509_21832_b200.runner.drive import snap_steps, steady_window
    plan = plan_time(t_final, cfl, mesh)
    n_steps = min(plan.n_steps, max_steps) if max_steps else plan.n_steps
    snaps = snap_steps(frame_times, plan.dt, n_steps)
    window = steady_window(n_steps)
    prob = oracle.Problem2D(mesh, bc, eps, model)
    frames, steady = [], 0.0
    for n in range(n_steps):
        Qp = Q
        Q, G, _ = oracle.step_2d_arrays(prob, Q, G, plan.dt)
        if track_steady and n >= n_steps - window:
            steady = max(steady, float(np.max(np.abs(Q - Qp))))
        if (n + 1) in snaps:
            H = oracle.heat_tensor_2d(G, Q[..., 1] / Q[..., 0], Q[..., 2] / Q[..., 0],
                                      prob.v1, prob.v2, eps)
            frames.append((snaps[n + 1], np.concatenate([np.moveaxis(Q, -1, 0), H])))
    return Q, G, frames, steady, n_steps


@pytest.mark.parametrize("name", ["step2d_box_walls", "step2d_wave_periodic"])
@pytest.mark.parametrize("max_steps", [None, 7])
def test_advance_matches_oracle_loop(mm, oracle, name, max_steps):
    from paper_2509_21832_b200.runner.drive import advance_2d
    mesh, bc, eps, model, p = problem_from_golden(name)
    d = np.load(GOLDEN / f"{name}.npz")
    t_final, cfl = 24 * float(d["dt"]), 0.4
    frame_times = (3 * float(d["dt"]), 3.2 * float(d["dt"]), 11 * float(d["dt"]), 99.0)
    snap = lambda st: mm.frame_moments(st, mesh, bc, eps, model)
    rec = advance_2d(mesh, bc, eps, model, mm.State2D(0.0, d["Q0"], d["G0"]), t_final, cfl,
                     frame_times=frame_times, max_steps=max_steps, snapshot=snap,
                     track_steady=True)
    Qo, Go, fo, steady_o, n_o = oracle_advance(oracle, mesh, bc, eps, model, d["Q0"], d["G0"],
                                               t_final, cfl, frame_times, max_steps, True)
    assert rec.steps_run == n_o
    assert rec.state.t == pytest.approx(n_o * rec.plan.dt, rel=1e-15)
    assert q_rel_err(rec.state.Q, Qo) <= 1e-9
    assert rel_err(rec.state.G, Go) <= 1e-10
    assert [t for t, _ in rec.frames] == [t for t, _ in fo]
    for (_, a), (_, b) in zip(rec.frames, fo):
        assert q_rel_err(np.moveaxis(a[:6], 0, -1), np.moveaxis(b[:6], 0, -1)) <= 1e-9
        assert rel_err(a[6:], b[6:]) <= 1e-9
    # steady change: a difference of nearby states, so an absolute bar on the Q scale
    assert abs(rec.steady_max_change - steady_o) <= 1e-10 * float(np.max(np.abs(Qo)))
    assert rec.steady_max_change > 0.0


def test_advance_source_path_matches_step_loop(mm):
    """With MMS sources the driver steps through step_2d; same result as the
    explicit loop, bitwise."""
    from test_oracle_golden import mms_problem
    from paper_2509_21832_b200.runner.drive import advance_2d
    mesh, bc, eps, model, exact, msrc, qsrc = mms_problem(8)
    Q0, G0 = exact(0.0)
    rec = advance_2d(mesh, bc, eps, model, mm.State2D(0.0, Q0, G0), 0.02, 0.926,
                     micro_source=msrc, macro_source=qsrc, track_steady=True)
    st = mm.State2D(0.0, Q0, G0)
    for n in range(rec.steps_run):
        st = mm.step_2d(st, mesh, bc, eps, model, rec.plan.dt, micro_source=msrc,
                        macro_source=qsrc)
        st.t = (n + 1) * rec.plan.dt
    assert np.array_equal(rec.state.Q, st.Q)
    assert np.array_equal(rec.state.G, st.G)
    assert np.isfinite(rec.steady_max_change) and rec.steady_max_change > 0

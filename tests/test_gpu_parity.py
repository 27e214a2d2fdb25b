"""GPU parity: the CUDA path (through the public API and the C ABI) against
the reference goldens and the CPU oracle.

Tolerances (north star, BASELINE.json): every conserved moment within 1e-11
relative L-inf after one step and 1e-9 after 100 steps (fp64).  The micro
field and the heat tensor are held to 1e-10 of their maxima.
"""

import numpy as np
import pytest

from conftest import (GOLDEN, golden_cases, golden_index, heat_sum_scale, prim_rel_err,
                      problem_from_golden, q_rel_err, rel_err)

pytestmark = pytest.mark.gpu

TOL_1 = 1e-11     # moments after one step
TOL_N = 1e-9      # moments after many steps
TOL_G = 1e-10     # micro field / heat tensor, relative to their maxima


@pytest.fixture(scope="module")
def mm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200 import _native
    _native.load()
    return mm


@pytest.mark.parametrize("name", golden_cases("step2d_"))
def test_step2d_matches_reference_goldens(mm, name):
    mesh, bc, eps, model, p = problem_from_golden(name)
    d = np.load(GOLDEN / f"{name}.npz")
    st = mm.State2D(0.0, d["Q0"], d["G0"])
    dt = float(d["dt"])
    for n in range(1, max(p["steps"]) + 1):
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
        if n in p["steps"]:
            tol = TOL_1 if n == 1 else TOL_N
            tg = TOL_G if n <= 10 else 1e-8
            assert q_rel_err(st.Q, d[f"Q{n}"]) <= tol, n
            assert prim_rel_err(st.Q, d[f"Q{n}"]) <= tol, n
            assert rel_err(st.G, d[f"G{n}"]) <= tg, n
            from paper_2509_21832_b200 import cell_centers
            hf = 1e-5 * heat_sum_scale(d[f"G{n}"], eps, cell_centers(mesh.velocity[0]),
                                       cell_centers(mesh.velocity[1]))
            assert rel_err(st.H_step.cpu().numpy(), d[f"Hstep{n}"], floor=hf) <= tg, n
            H = mm.frame_moments(st, mesh, bc, eps, model)[6:]
            assert rel_err(H, d[f"Hframe{n}"], floor=hf) <= tg, n


def _random_problem(mm, nx, ny, nv, faces, nu, eps, seed, kind="esbgk_2d"):
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, PhaseMesh,
                                       conserved_2d)
    rng = np.random.default_rng(seed)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, nx), Axis(0.0, 1.0, ny)),
                     velocity=(Axis(-7.0, 7.0, nv), Axis(-7.0, 7.0, nv)))
    bc = BoundarySpec2D(*faces)
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y, indexing="ij")
    ph = rng.uniform(0, 2 * np.pi, 6)
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * X + ph[0]) * np.cos(2 * np.pi * Y + ph[1])
    u1 = 0.3 * np.cos(2 * np.pi * Y + ph[2])
    u2 = -0.2 * np.sin(2 * np.pi * X + ph[3])
    t11 = 1.0 + 0.1 * np.cos(2 * np.pi * X + ph[4])
    t22 = 1.0 + 0.1 * np.sin(2 * np.pi * Y + ph[5])
    t12 = 0.05 * np.sin(2 * np.pi * (X + Y))
    Q = conserved_2d(rho, u1, u2, t11, t12, t22)
    G = 0.01 * rng.standard_normal((nx, ny, nv, nv))
    model = CollisionModel(kind, nu=nu)
    dt = 0.4 * min(1.0 / nx, 1.0 / ny) / 7.0
    return mesh, bc, eps, model, Q, G, dt


@pytest.mark.parametrize("faces_kind", ["periodic", "extrapolate", "walls"])
def test_v1024_vs_oracle_1_and_100_steps(mm, oracle, faces_kind):
    """The benchmark velocity grid (32 x 32) on a 24 x 20 spatial grid:
    1e-11 after one step, 1e-9 after 100 steps, against the C oracle."""
    from paper_2509_21832_b200 import EXTRAPOLATE, PERIODIC, WallSpec
    faces = {"periodic": (PERIODIC,) * 4, "extrapolate": (EXTRAPOLATE,) * 4,
             "walls": (WallSpec(1.0), WallSpec(1.0), WallSpec(1.0), WallSpec(1.0, 0.16))}[faces_kind]
    mesh, bc, eps, model, Q, G, dt = _random_problem(mm, 24, 20, 32, faces, -0.5, 0.05, 7)
    prob = oracle.Problem2D(mesh, bc, eps, model)
    st = mm.State2D(0.0, Q, G)
    Qo, Go = Q, G
    for n in range(1, 101):
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
        Qo, Go, _ = oracle.step_2d_arrays(prob, Qo, Go, dt)
        if n == 1:
            assert q_rel_err(st.Q, Qo) <= TOL_1
            assert rel_err(st.G, Go) <= TOL_G
    assert q_rel_err(st.Q, Qo) <= TOL_N
    assert rel_err(st.G, Go) <= 1e-8


def test_graph_run_equals_step_loop(mm):
    """run_2d (one CUDA-graph replay) is bitwise the step_2d loop."""
    from paper_2509_21832_b200 import PERIODIC, cell_centers, plan_time
    mesh, bc, eps, model, Q, G, dt = _random_problem(mm, 16, 16, 32, (PERIODIC,) * 4, -0.5,
                                                      0.1, 3)
    solver = mm.get_solver(mesh, bc, eps, model)
    import torch
    Qd = torch.from_numpy(Q).cuda()
    Gd = torch.from_numpy(G).cuda()
    Qa, Ga = solver.run(Qd.clone(), Gd.clone(), dt, 7)
    st = mm.State2D(0.0, Q, G)
    for _ in range(7):
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
    assert np.array_equal(Qa.cpu().numpy(), st.Q)
    assert np.array_equal(Ga.cpu().numpy(), st.G)


def test_run_2d_matches_oracle(mm, oracle):
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, EXTRAPOLATE,
                                       PhaseMesh, plan_time)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, 16), Axis(0.0, 1.0, 16)),
                     velocity=(Axis(-8.0, 8.0, 16), Axis(-8.0, 8.0, 16)))
    bc = BoundarySpec2D(EXTRAPOLATE, EXTRAPOLATE, EXTRAPOLATE, EXTRAPOLATE)
    model = CollisionModel("esbgk_2d", nu=-0.5)
    x = (np.arange(16) + 0.5) / 16
    X, Y = np.meshgrid(x, x, indexing="ij")
    rho = np.where(Y >= 0.5, np.where(X >= 0.5, 1.0, 0.5), np.where(X >= 0.5, 0.5, 0.25))
    u1 = np.where(X >= 0.5, 0.0, 0.5)
    u2 = np.where(Y >= 0.5, 0.0, 0.5)
    T = np.where(Y >= 0.5, np.where(X >= 0.5, 1.0, 0.8), np.where(X >= 0.5, 0.8, 0.6))
    G0 = np.zeros((16, 16, 16, 16))
    st, plan = mm.run_2d(mesh, bc, 1e-2, model, rho, u1, u2, T, 0 * T, T, G0, 0.02, 0.4)
    from paper_2509_21832_b200 import conserved_2d
    prob = oracle.Problem2D(mesh, bc, 1e-2, model)
    Qo, Go, _ = oracle.run_steps_2d(prob, conserved_2d(rho, u1, u2, T, 0 * T, T), G0,
                                    plan.dt, plan.n_steps)
    assert st.t == pytest.approx(0.02)
    assert q_rel_err(st.Q, Qo) <= TOL_N


@pytest.mark.parametrize("case", ["density", "pressure_spd", "pressure_t11", "density_and_spd"])
def test_invalid_state_reports_reference_cell(mm, case):
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, PERIODIC,
                                       PhaseMesh)
    want = golden_index()["errors"][case]
    Q = np.load(GOLDEN / f"err_{case}_Q.npy")
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, 6), Axis(0.0, 1.0, 5)),
                     velocity=(Axis(-5.0, 5.0, 6), Axis(-5.0, 5.0, 6)))
    bc = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
    model = CollisionModel("esbgk_2d", nu=-0.5)
    st = mm.State2D(0.0, Q, np.zeros((6, 5, 6, 6)))
    st = mm.step_2d(st, mesh, bc, 0.1, model, 1e-3)
    with pytest.raises(mm.InvalidStateError) as ei:
        _ = st.Q
    assert list(ei.value.cell) == want["cell"]
    assert ei.value.value == pytest.approx(want["value"], rel=1e-14)


def test_kernel_contract_matches_reference(mm):
    """The ten plugin kernels vs the reference's compiled kernels
    (1e-12 * max|ref|, the reference's own cross-backend bar)."""
    from paper_2509_21832_b200 import _kernels as K
    k = np.load(GOLDEN / "kernels.npz")
    v1, v2 = k["v1"], k["v2"]
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    M = K.maxwellian_field_2d(k["rho"], k["u1"], k["u2"], k["T"], v1, v2)
    assert rel_err(M, k["maxwellian"]) <= 1e-12
    M = k["maxwellian"]
    args = (k["rho"], k["u1"], k["u2"], k["T"], v1, v2)
    assert rel_err(K.project_field_2d(k["G"], M, *args, dv), k["project"]) <= 1e-12
    assert rel_err(K.transport_stage_2d(k["Gx"], M, *args, 0.02, 0.003, 0), k["transport0"]) <= 1e-12
    assert rel_err(K.transport_stage_2d(k["Gy"], M, *args, 0.02, 0.003, 1), k["transport1"]) <= 1e-12
    gh = K.ghat_2d(M, k["rho"], k["u1"], k["u2"], k["T"], k["s11"], k["s12"], k["g1"], k["g2"],
                   k["tau"], v1, v2)
    assert rel_err(gh, k["ghat"]) <= 1e-12
    a = np.array(k["G"], copy=True)
    K.add_gaussian_term_2d(a, M, k["rho"], k["u1"], k["u2"], k["m11"], k["m12"], k["m22"], 0.07,
                           v1, v2)
    assert rel_err(a, k["gauss"]) <= 1e-12
    a = np.array(k["G"], copy=True)
    K.add_lowrank_4d(a, k["coeffs"], k["shapes"])
    assert rel_err(a, k["lowrank"]) <= 1e-12
    assert rel_err(K.relax_2d(k["G"], k["Ghat"], k["tau"], 0.004, 0.08), k["relax"]) <= 1e-12
    H = K.heat_tensor_2d(k["G"], k["u1"], k["u2"], v1, v2, dv, 0.08)
    for x, y in zip(H, k["heat"]):
        assert rel_err(x, y) <= 1e-12
    assert rel_err(K.upwind_z_1d(k["G1x"], k["v"], 0.05), k["upwind1d"]) <= 1e-12
    v40 = k["v40"]
    assert rel_err(K.project_field_1d(k["F1"], k["M1"], k["rho1"], k["uu"], k["T1"], v40,
                                      v40[1] - v40[0]), k["project1d"]) <= 1e-12


def test_mms_regression_pin_on_gpu(mm):
    """The reference's frozen mms_run_2d(20) errors (test_cases.py:104-107)
    reproduced by the GPU step with the manufactured sources."""
    from test_oracle_golden import mms_problem, relative_l2
    from paper_2509_21832_b200 import plan_time
    mesh, bc, eps, model, exact, msrc, qsrc = mms_problem(20)
    plan = plan_time(0.25, 0.926, mesh)
    Q, G = exact(0.0)
    st = mm.State2D(0.0, Q, G)
    for n in range(plan.n_steps):
        st = mm.step_2d(st, mesh, bc, eps, model, plan.dt, micro_source=msrc, macro_source=qsrc)
        st.t = (n + 1) * plan.dt
    Qe, Ge = exact(0.25)
    assert relative_l2(st.Q, Qe) == pytest.approx(0.030605594996427687, rel=1e-10)
    assert relative_l2(st.G, Ge) == pytest.approx(0.031135911051471035, rel=1e-10)


def test_full_size_c2_conservation(mm):
    """C2 at full size (256^2 x 32^2, periodic): mass, momentum and the
    energy trace are conserved to roundoff over 20 steps (size-independent
    property; the oracle is too slow at this size for 100 steps)."""
    import torch
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, PERIODIC,
                                       PhaseMesh, conserved_2d)
    n = 256
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, n), Axis(0.0, 1.0, n)),
                     velocity=(Axis(-7.0, 7.0, 32), Axis(-7.0, 7.0, 32)))
    bc = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
    model = CollisionModel("esbgk_2d", nu=-0.5)
    x = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(x, x, indexing="ij")
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)
    Q = conserved_2d(rho, 0.5, 0.5, 1.0, 0.0, 1.0)
    solver = mm.get_solver(mesh, bc, 0.1, model)
    Qd = torch.from_numpy(Q).cuda()
    Gd = torch.zeros((n, n, 32, 32), dtype=torch.float64, device="cuda")
    dt = 0.4 * (1.0 / n) / 7.0
    Qf, Gf = solver.run(Qd, Gd, dt, 20)
    solver.check()
    Qf = Qf.cpu().numpy()
    inv0 = [Q[..., 0].sum(), Q[..., 1].sum(), Q[..., 2].sum(), (Q[..., 3] + Q[..., 5]).sum()]
    inv1 = [Qf[..., 0].sum(), Qf[..., 1].sum(), Qf[..., 2].sum(), (Qf[..., 3] + Qf[..., 5]).sum()]
    for a, b in zip(inv0, inv1):
        assert abs(a - b) <= 1e-11 * abs(a)


# -- block decomposition (reference test_parallel.py:96-128) ---------------

def _parallel_problem(nx, ny, nv, faces, seed):
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, PhaseMesh,
                                       conserved_2d)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, nx), Axis(0.0, 1.0, ny)),
                     velocity=(Axis(-5.0, 5.0, nv), Axis(-5.0, 5.0, nv)))
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y, indexing="ij")
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)
    T = 1.0 + 0.1 * np.cos(2 * np.pi * X)
    Q = conserved_2d(rho, 0.02 * np.cos(2 * np.pi * Y), -0.03 * np.sin(2 * np.pi * X), T,
                     0.02 * np.sin(2 * np.pi * (X + Y)), T)
    G = 0.01 * np.random.default_rng(seed).standard_normal((nx, ny, nv, nv))
    return mesh, BoundarySpec2D(*faces), CollisionModel("esbgk_2d", nu=-0.5), Q, G


@pytest.mark.parametrize("halo", ["peer", "packed"])
@pytest.mark.parametrize("nv", [6, 32])
@pytest.mark.parametrize("grid,faces", [
    ((2, 2), "cavity"), ((3, 4), "cavity"), ((2, 2), "periodic"), ((4, 3), "mixed"),
    ((1, 1), "periodic"), ((2, 1), "periodic"), ((1, 3), "cavity"), ((3, 2), "periodic"),
    ((1, 2), "periodic")])
def test_block_grid_equals_serial_bitwise(mm, grid, faces, nv, halo):
    """Both forms of the G halo: "peer" (ghost cells read in place from the
    neighbour blocks' arrays) and "packed" (pack, copy, receive)."""
    from paper_2509_21832_b200 import EXTRAPOLATE, PERIODIC, WallSpec
    from paper_2509_21832_b200.parallel import run_parallel_2d
    w = WallSpec(1.0)
    fc = {"cavity": (w, w, w, WallSpec(1.0, 0.16)), "periodic": (PERIODIC,) * 4,
          "mixed": (EXTRAPOLATE, EXTRAPOLATE, PERIODIC, PERIODIC)}[faces]
    mesh, bc, model, Q0, G0 = _parallel_problem(12, 12, nv, fc, 11)
    dt = 0.3 * (1.0 / 12) / 5.0
    Qp, Gp, _, _ = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, dt, 6, grid=grid, halo=halo)
    st = mm.State2D(0.0, Q0, G0)
    for _ in range(6):
        st = mm.step_2d(st, mesh, bc, 0.08, model, dt)
    assert np.array_equal(Qp, st.Q)
    assert np.array_equal(Gp, st.G)


@pytest.mark.parametrize("halo", ["peer", "packed"])
@pytest.mark.parametrize("nsteps", [1, 5])
def test_block_grid_graph_replay_equals_eager(mm, nsteps, halo):
    """run_parallel_2d's CUDA-graph replay of the decomposed step (blocks on
    one GPU) is bitwise its eager issue and the serial step, for an odd step
    count too (the ping-pong parity)."""
    from paper_2509_21832_b200 import PERIODIC, WallSpec
    from paper_2509_21832_b200.parallel import run_parallel_2d
    w = WallSpec(1.0)
    mesh, bc, model, Q0, G0 = _parallel_problem(12, 12, 32, (PERIODIC, PERIODIC, w, w), 5)
    dt = 0.3 * (1.0 / 12) / 5.0
    Qg, Gg, _, _ = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, dt, nsteps, grid=(2, 3),
                                   halo=halo)
    Qe, Ge, _, _ = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, dt, nsteps, grid=(2, 3),
                                   graph=False, halo=halo)
    st = mm.State2D(0.0, Q0, G0)
    for _ in range(nsteps):
        st = mm.step_2d(st, mesh, bc, 0.08, model, dt)
    assert np.array_equal(Qg, Qe) and np.array_equal(Gg, Ge)
    assert np.array_equal(Qg, st.Q) and np.array_equal(Gg, st.G)


def test_block_grid_steady_tracking(mm):
    from paper_2509_21832_b200 import PERIODIC
    from paper_2509_21832_b200.parallel import run_parallel_2d
    mesh, bc, model, Q0, G0 = _parallel_problem(8, 8, 6, (PERIODIC,) * 4, 3)
    Q, G, smax, secs = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, 1e-3, 4, grid=(2, 2),
                                       track_from=2)
    assert np.isfinite(smax) and smax > 0.0 and secs > 0.0
    _, _, snan, _ = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, 1e-3, 2, grid=(2, 2))
    assert np.isnan(snan)


@pytest.mark.parametrize("shape", [(1, 7), (7, 1), (2, 2), (1, 1), (3, 50)])
@pytest.mark.parametrize("faces_kind", ["periodic", "walls", "extrapolate"])
def test_v1024_degenerate_grids_vs_oracle(mm, oracle, shape, faces_kind):
    """The 32 x 32 kernel on degenerate spatial grids (a single column or
    row, one cell, a band shorter than ly, ly + 2 rows): each cell's own
    neighbour is itself under wrap, walls meet at corners.  10 steps."""
    from paper_2509_21832_b200 import EXTRAPOLATE, PERIODIC, WallSpec
    faces = {"periodic": (PERIODIC,) * 4, "extrapolate": (EXTRAPOLATE,) * 4,
             "walls": (WallSpec(1.0), WallSpec(0.9), WallSpec(1.1), WallSpec(1.0, 0.2))}[faces_kind]
    nx, ny = shape
    mesh, bc, eps, model, Q, G, dt = _random_problem(mm, nx, ny, 32, faces, -0.5, 0.05, 11)
    prob = oracle.Problem2D(mesh, bc, eps, model)
    st = mm.State2D(0.0, Q, G)
    Qo, Go = Q, G
    for n in range(1, 11):
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
        Qo, Go, _ = oracle.step_2d_arrays(prob, Qo, Go, dt)
    assert q_rel_err(st.Q, Qo) <= TOL_N
    # a lone periodic cell relaxes G to ~1e-6, pure roundoff of the O(0.1)
    # Maxwellian terms: compare G on a 1e-4 floor
    assert rel_err(st.G, Go, floor=1e-4) <= TOL_G


# -- band layouts of the 32 x 32 kernel (mm2d_api.cu pick_bands) ----------

@pytest.mark.parametrize("bands", ["auto", "7,20,5", "1,1,30", "32", "3,3,3,3,3,3,3,11"])
def test_v1024_band_layout_is_bitwise_neutral(mm, bands, monkeypatch):
    """The specialised kernel walks each column in bands of rows; the layout
    (uniform, the automatic long/short split, or explicit MM2D_BANDS) only
    changes the schedule, never the arithmetic: results are bitwise equal."""
    import torch
    from paper_2509_21832_b200 import PERIODIC, WallSpec
    from paper_2509_21832_b200.solver import Solver2D
    w = WallSpec(1.0)
    mesh, bc, eps, model, Q, G, dt = _random_problem(mm, 9, 32, 32, (w, w, PERIODIC, PERIODIC),
                                                     -0.5, 0.05, 5)
    outs = []
    for env in ({"MM2D_LY": "32"}, {} if bands == "auto" else {"MM2D_BANDS": bands}):
        for k in ("MM2D_LY", "MM2D_BANDS"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = Solver2D(mesh, bc, eps, model)
        Qd = torch.from_numpy(Q).cuda()
        Gd = torch.from_numpy(G).cuda()
        for _ in range(3):
            Qd, Gd, Hd = s.step(Qd, Gd, dt)
        torch.cuda.synchronize()
        s.check()
        outs.append((Qd.cpu().numpy(), Gd.cpu().numpy(), Hd.cpu().numpy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("halo", ["packed", "peer"])
@pytest.mark.parametrize("nv", [6, 32])
@pytest.mark.parametrize("faces,eps", [("periodic", 0.08), ("mixed", 0.08), ("periodic", 1e-12)])
def test_block_grid_overlap_split_equals_serial(mm, faces, eps, nv, halo):
    """Blocks tall and wide enough that every split has interior micro CTAs
    (run while the G halo is in flight) and perimeter CTAs (a separate
    launch on a side stream): the decomposed step stays bitwise the serial
    one, also at eps < 1e-10 where every micro launch reads the isotropy
    maxima the prep accumulates."""
    from paper_2509_21832_b200 import EXTRAPOLATE, PERIODIC
    from paper_2509_21832_b200.parallel import run_parallel_2d
    fc = {"periodic": (PERIODIC,) * 4,
          "mixed": (EXTRAPOLATE, EXTRAPOLATE, PERIODIC, PERIODIC)}[faces]
    mesh, bc, model, Q0, G0 = _parallel_problem(24, 400, nv, fc, 13)
    dt = 0.3 * (1.0 / 400) / 5.0
    Qp, Gp, _, _ = run_parallel_2d(mesh, bc, eps, model, Q0, G0, dt, 3, grid=(2, 2), halo=halo)
    st = mm.State2D(0.0, Q0, G0)
    for _ in range(3):
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
    assert np.array_equal(Qp, st.Q)
    assert np.array_equal(Gp, st.G)

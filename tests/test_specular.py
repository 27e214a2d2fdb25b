"""Specular (reflecting) walls -- an extension beyond the reference, which has
only diffuse walls (BASELINE config 4 asks for reflecting walls; SURVEY
§8(f) row f4).

There is no reference implementation to pin against, so the rule is pinned by
the method of images instead: a specular box [0, 1]^2 must evolve exactly
like the periodic box [0, 2]^2 holding the box and its mirror images
(f(2 - x, y, -v1, v2) and f(x, 2 - y, v1, -v2)), restricted to [0, 1]^2.  The
periodic path is itself pinned to the reference goldens
(test_oracle_golden.py, test_gpu_parity.py), so the image identity pins the
specular ghosts to roundoff (only per-cell summation orders differ).

CPU tests: the oracle against the images and its conservation properties,
host validation.  GPU tests: the CUDA path against the oracle (1 and 100
steps at the north-star tolerances), against the images, mixed with diffuse
walls and in a block decomposition (bitwise equal to the serial step).
"""

import numpy as np
import pytest

from conftest import q_rel_err, rel_err

NV = 16


def _state(nx, ny, nv, seed=3, amp=1e-3):
    import paper_2509_21832_b200 as mm
    rng = np.random.default_rng(seed)
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y, indexing="ij")
    rho = 1 + 0.3 * np.exp(-((X - 0.3) ** 2 + (Y - 0.6) ** 2) / 0.02)
    u1 = 0.2 * np.sin(2 * np.pi * X) * np.cos(np.pi * Y)
    u2 = 0.1 * np.sin(np.pi * X) * np.sin(2 * np.pi * Y)
    T = 1 + 0.1 * np.cos(np.pi * X)
    Q = mm.conserved_2d(rho, u1, u2, T, 0.02 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y),
                        T * 1.01)
    G = amp * rng.standard_normal((nx, ny, nv, nv))
    return Q, G


def _image_x(Q, G):
    Qm = Q[::-1].copy()
    Qm[..., 1] *= -1
    Qm[..., 4] *= -1
    return np.concatenate([Q, Qm], 0), np.concatenate([G, G[::-1, :, ::-1, :]], 0)


def _image_y(Q, G):
    Qm = Q[:, ::-1].copy()
    Qm[..., 2] *= -1
    Qm[..., 4] *= -1
    return np.concatenate([Q, Qm], 1), np.concatenate([G, G[:, ::-1, :, ::-1]], 1)


def _problem(nx, ny, faces, nv=NV, vmax=8.0, lx=1.0, ly=1.0):
    import paper_2509_21832_b200 as mm
    mesh = mm.PhaseMesh(space=(mm.Axis(0, lx, nx), mm.Axis(0, ly, ny)),
                        velocity=(mm.Axis(-vmax, vmax, nv), mm.Axis(-vmax, vmax, nv)))
    return mesh, mm.BoundarySpec2D(*faces), mm.CollisionModel("esbgk_2d", nu=-0.5)


def _run(stepper, Q, G, n):
    for _ in range(n):
        Q, G, H = stepper(Q, G)
    return Q, G, H


# ---------------------------------------------------------------- CPU ----

def test_oracle_specular_box_equals_periodic_images(oracle):
    import paper_2509_21832_b200 as mm
    n, eps = 12, 0.05
    dt = 0.4 * (1 / n) / 8
    Q, G = _state(n, n, NV)
    mesh, bc, model = _problem(n, n, (mm.SPECULAR,) * 4)
    p = oracle.Problem2D(mesh, bc, eps, model)
    Qs, Gs, Hs = _run(lambda q, g: oracle.step_2d_arrays(p, q, g, dt), Q, G, 5)
    Q2, G2 = _image_y(*_image_x(Q, G))
    mesh2, bc2, _ = _problem(2 * n, 2 * n, (mm.PERIODIC,) * 4, lx=2.0, ly=2.0)
    p2 = oracle.Problem2D(mesh2, bc2, eps, model)
    Q2, G2, H2 = _run(lambda q, g: oracle.step_2d_arrays(p2, q, g, dt), Q2, G2, 5)
    assert q_rel_err(Qs, Q2[:n, :n]) <= 1e-14
    assert rel_err(Gs, G2[:n, :n]) <= 1e-13
    assert rel_err(Hs, H2[:, :n, :n]) <= 1e-13


def test_oracle_specular_x_only_equals_images(oracle):
    import paper_2509_21832_b200 as mm
    nx, ny, eps = 10, 6, 0.02
    dt = 0.4 * (1 / nx) / 8
    Q, G = _state(nx, ny, NV, seed=5)
    mesh, bc, model = _problem(nx, ny, (mm.SPECULAR, mm.SPECULAR, mm.PERIODIC, mm.PERIODIC))
    p = oracle.Problem2D(mesh, bc, eps, model)
    Qs, Gs, _ = _run(lambda q, g: oracle.step_2d_arrays(p, q, g, dt), Q, G, 4)
    Q2, G2 = _image_x(Q, G)
    mesh2, bc2, _ = _problem(2 * nx, ny, (mm.PERIODIC,) * 4, lx=2.0)
    p2 = oracle.Problem2D(mesh2, bc2, eps, model)
    Q2, G2, _ = _run(lambda q, g: oracle.step_2d_arrays(p2, q, g, dt), Q2, G2, 4)
    assert q_rel_err(Qs, Q2[:nx]) <= 1e-14
    assert rel_err(Gs, G2[:nx]) <= 1e-13


def test_oracle_specular_box_conserves_mass_and_energy(oracle):
    """Closed box: zero mass flux through every wall; the energy trace is
    conserved by the KFVS fluxes and the heat sources (interface heat of
    the odd components vanishes at the wall)."""
    import paper_2509_21832_b200 as mm
    n = 10
    Q, G = _state(n, n, NV, amp=0.0)
    mesh, bc, model = _problem(n, n, (mm.SPECULAR,) * 4)
    p = oracle.Problem2D(mesh, bc, 0.05, model)
    Qs, _, _ = _run(lambda q, g: oracle.step_2d_arrays(p, q, g, 0.4 * (1 / n) / 8), Q, G, 20)
    m0, m1 = Q[..., 0].sum(), Qs[..., 0].sum()
    e0, e1 = (Q[..., 3] + Q[..., 5]).sum(), (Qs[..., 3] + Qs[..., 5]).sum()
    assert abs(m1 - m0) <= 1e-13 * m0
    assert abs(e1 - e0) <= 1e-12 * e0


def test_specular_is_2d_only():
    import paper_2509_21832_b200 as mm
    with pytest.raises(mm.ConfigurationError):
        mm.BoundarySpec1D(mm.SPECULAR, mm.SPECULAR)
    bc = mm.BoundarySpec2D(mm.SPECULAR, mm.SPECULAR, mm.PERIODIC, mm.PERIODIC)
    from paper_2509_21832_b200.boundary import face_code
    assert [face_code(f) for f in bc.faces] == [3, 3, 0, 0]
    with pytest.raises(mm.ConfigurationError):   # periodic faces still pair
        mm.BoundarySpec2D(mm.SPECULAR, mm.PERIODIC, mm.PERIODIC, mm.PERIODIC)


# ---------------------------------------------------------------- GPU ----

@pytest.fixture(scope="module")
def mm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200 import _native
    _native.load()
    return mm


def _gpu_stepper(mm, mesh, bc, eps, model, dt):
    holder = {}

    def step(Q, G):
        st = holder.get("st") or mm.State2D(0.0, Q, G)
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
        holder["st"] = st
        return st.Q, st.G, st.H_step.cpu().numpy()
    return step


@pytest.mark.gpu
@pytest.mark.parametrize("nv", [32, 12])
@pytest.mark.parametrize("faces", ["box", "x_only", "y_only", "mixed_diffuse"])
def test_gpu_specular_vs_oracle(mm, oracle, nv, faces):
    """nv = 32: the specialised 32 x 32 kernel; nv = 12: the generic kernel.
    North-star tolerances: 1e-11 after 1 step, 1e-9 after 100 steps."""
    S, P, W = mm.SPECULAR, mm.PERIODIC, mm.WallSpec
    fc = {"box": (S, S, S, S), "x_only": (S, S, P, P), "y_only": (P, P, S, S),
          "mixed_diffuse": (S, S, W(1.0), W(1.0, 0.2))}[faces]
    nx, ny, eps = 20, 18, 0.05
    mesh, bc, model = _problem(nx, ny, fc, nv=nv)
    dt = 0.4 * (1 / nx) / 8
    Q, G = _state(nx, ny, nv, seed=7, amp=1e-2)
    prob = oracle.Problem2D(mesh, bc, eps, model)
    st = mm.State2D(0.0, Q, G)
    Qo, Go = Q, G
    for n in range(1, 101):
        st = mm.step_2d(st, mesh, bc, eps, model, dt)
        Qo, Go, Ho = oracle.step_2d_arrays(prob, Qo, Go, dt)
        if n == 1:
            assert q_rel_err(st.Q, Qo) <= 1e-11
            assert rel_err(st.G, Go) <= 1e-10
            assert rel_err(st.H_step.cpu().numpy(), Ho) <= 1e-10
    assert q_rel_err(st.Q, Qo) <= 1e-9
    assert rel_err(st.G, Go) <= 1e-8


@pytest.mark.gpu
def test_gpu_specular_box_equals_periodic_images(mm):
    """The 32 x 32 kernel: specular box == periodic images (both on the GPU)."""
    n, eps = 16, 0.05
    dt = 0.4 * (1 / n) / 8
    Q, G = _state(n, n, 32, amp=1e-2)
    mesh, bc, model = _problem(n, n, (mm.SPECULAR,) * 4, nv=32)
    Qs, Gs, Hs = _run(_gpu_stepper(mm, mesh, bc, eps, model, dt), Q, G, 10)
    Q2, G2 = _image_y(*_image_x(Q, G))
    mesh2, bc2, _ = _problem(2 * n, 2 * n, (mm.PERIODIC,) * 4, nv=32, lx=2.0, ly=2.0)
    Q2, G2, H2 = _run(_gpu_stepper(mm, mesh2, bc2, eps, model, dt), Q2, G2, 10)
    assert q_rel_err(Qs, Q2[:n, :n]) <= 1e-13
    assert rel_err(Gs, G2[:n, :n]) <= 1e-12
    assert rel_err(Hs, H2[:, :n, :n]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("nv", [6, 32])
@pytest.mark.parametrize("grid", [(2, 2), (3, 2), (1, 3)])
def test_gpu_specular_block_grid_equals_serial_bitwise(mm, grid, nv):
    from paper_2509_21832_b200.parallel import run_parallel_2d
    S = mm.SPECULAR
    n = 12
    mesh, bc, model = _problem(n, n, (S, S, S, mm.WallSpec(1.0, 0.16)), nv=nv, vmax=5.0)
    Q0, G0 = _state(n, n, nv, seed=11, amp=1e-2)
    dt = 0.3 * (1.0 / n) / 5.0
    Qp, Gp, _, _ = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, dt, 6, grid=grid)
    st = mm.State2D(0.0, Q0, G0)
    for _ in range(6):
        st = mm.step_2d(st, mesh, bc, 0.08, model, dt)
    assert np.array_equal(Qp, st.Q)
    assert np.array_equal(Gp, st.G)


@pytest.mark.gpu
@pytest.mark.parametrize("halo", ["packed", "peer"])
@pytest.mark.parametrize("nv", [6, 32])
def test_gpu_specular_overlap_split_equals_serial(mm, nv, halo):
    """Blocks large enough that the split micro launch has interior CTAs
    (run while the G halo is in flight) and perimeter CTAs, with specular
    faces on the physical boundary: still bitwise the serial step."""
    from paper_2509_21832_b200.parallel import run_parallel_2d
    S = mm.SPECULAR
    nx, ny = 24, 400
    mesh, bc, model = _problem(nx, ny, (S, S, S, S), nv=nv, vmax=5.0)
    Q0, G0 = _state(nx, ny, nv, seed=12, amp=1e-2)
    dt = 0.3 * (1.0 / ny) / 5.0
    Qp, Gp, _, _ = run_parallel_2d(mesh, bc, 0.08, model, Q0, G0, dt, 3, grid=(2, 2), halo=halo)
    st = mm.State2D(0.0, Q0, G0)
    for _ in range(3):
        st = mm.step_2d(st, mesh, bc, 0.08, model, dt)
    assert np.array_equal(Qp, st.Q)
    assert np.array_equal(Gp, st.G)


@pytest.mark.gpu
def test_gpu_specular_needs_symmetric_velocity_axis(mm):
    mesh = mm.PhaseMesh(space=(mm.Axis(0, 1, 4), mm.Axis(0, 1, 4)),
                        velocity=(mm.Axis(-6.0, 7.0, 12), mm.Axis(-7.0, 7.0, 12)))
    Q, G = _state(4, 4, 12)
    bc = mm.BoundarySpec2D(mm.SPECULAR, mm.SPECULAR, mm.PERIODIC, mm.PERIODIC)
    with pytest.raises(mm.ConfigurationError):
        mm.step_2d(mm.State2D(0.0, Q, G), mesh, bc, 0.05, mm.CollisionModel("esbgk_2d"), 1e-3)
    # only the wall-normal axis has to be symmetric
    bc = mm.BoundarySpec2D(mm.PERIODIC, mm.PERIODIC, mm.SPECULAR, mm.SPECULAR)
    st = mm.step_2d(mm.State2D(0.0, Q, G), mesh, bc, 0.05, mm.CollisionModel("esbgk_2d"), 1e-3)
    assert np.isfinite(st.Q).all()

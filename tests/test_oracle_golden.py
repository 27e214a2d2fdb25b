"""Pin the CPU oracle to the reference itself.

The fixtures in tests/golden/ were produced by running the reference solver
(compiled backend) with tests/golden/make_golden.py.  The oracle must
reproduce them to a few ulps, which is what makes it a trustworthy checker
for the CUDA path (tests/test_gpu_parity.py).
"""

import math

import numpy as np
import pytest

from conftest import (GOLDEN, golden_cases, golden_index, h_rel_err, prim_rel_err,
                      problem_from_golden, q_rel_err, rel_err)


@pytest.mark.parametrize("name", golden_cases("step2d_"))
def test_oracle_matches_reference_step2d(oracle, name):
    mesh, bc, eps, model, p = problem_from_golden(name)
    d = np.load(GOLDEN / f"{name}.npz")
    prob = oracle.Problem2D(mesh, bc, eps, model)
    Q, G = d["Q0"], d["G0"]
    for n in range(1, max(p["steps"]) + 1):
        Q, G, H = oracle.step_2d_arrays(prob, Q, G, float(d["dt"]))
        if n in p["steps"]:
            tol = 1e-13 if n == 1 else 1e-11
            assert q_rel_err(Q, d[f"Q{n}"]) <= tol
            assert prim_rel_err(Q, d[f"Q{n}"]) <= tol
            assert rel_err(G, d[f"G{n}"]) <= 1e-11
            assert rel_err(H, d[f"Hstep{n}"]) <= 1e-11
            Hf = oracle.heat_tensor_2d(G, Q[..., 1] / Q[..., 0], Q[..., 2] / Q[..., 0],
                                       prob.v1, prob.v2, eps)
            assert rel_err(Hf, d[f"Hframe{n}"]) <= 1e-11


def config_problem(name, mm=None):
    """bench.py's workload for a cfg_* golden (the generator the fixture was
    made with), as this repo's host-side problem objects."""
    import bench
    p = golden_index()[name]
    eps = p["eps"] if p["config"] == "c3" else None
    return bench.make_workload(p["config"], n=p["n"], eps=eps, seed=p["seed"]), p


@pytest.mark.parametrize("name", golden_cases("cfg_"))
def test_bench_generators_reproduce_golden_inputs(name):
    """bench.py builds exactly the initial state the reference was run on."""
    cfg, p = config_problem(name)
    d = np.load(GOLDEN / f"{name}.npz")
    assert np.array_equal(cfg["initial"](0, p["n"], 0, p["n"]), d["Q0"])
    assert cfg["dt"] == float(d["dt"])


@pytest.mark.parametrize("name", golden_cases("cfg_"))
def test_oracle_matches_reference_configs(oracle, name):
    """The BASELINE configurations as bench.py builds them (12^2 cells,
    32^2 velocities), 100 steps: moments, primitives and heat tensors."""
    cfg, p = config_problem(name)
    d = np.load(GOLDEN / f"{name}.npz")
    prob = oracle.Problem2D(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"])
    Q, G = d["Q0"], np.zeros((p["n"], p["n"], 32, 32))
    for n in range(1, 101):
        Qn, G, H = oracle.step_2d_arrays(prob, Q, G, cfg["dt"])
        if n in (1, 10, 100):
            tol = 1e-13 if n == 1 else 1e-11
            assert q_rel_err(Qn, d[f"Q{n}"]) <= tol, n
            assert prim_rel_err(Qn, d[f"Q{n}"]) <= tol, n
            assert h_rel_err(H, d[f"Hstep{n}"], d[f"Q{n}"], cfg["eps"]) <= 1e-10, n
        Q = Qn
    if "G100" in d.files:
        assert rel_err(G, d["G100"]) <= 1e-10


@pytest.mark.parametrize("name", golden_cases("step1d_"))
def test_oracle_matches_reference_step1d(oracle, name):
    from types import SimpleNamespace as NS
    p = golden_index()[name]
    d = np.load(GOLDEN / f"{name}.npz")
    mesh = NS(space=(NS(min=0.0, max=1.0, n=p["nx"]),),
              velocity=(NS(min=p["v"][0], max=p["v"][1], n=p["v"][2]),))

    def face(f):
        return NS(temperature=f["wall"]) if isinstance(f, dict) else f

    bc = NS(left=face(p["faces"][0]), right=face(p["faces"][1]))
    model = NS(kind=p["kind"], nu=0.0, value=1.0)
    prob = oracle.Problem1D(mesh, bc, p["eps"], model)
    Q, G = d["Q0"], d["G0"]
    for n in range(1, max(p["steps"]) + 1):
        Q, G, _ = oracle.step_1d_arrays(prob, Q, G, float(d["dt"]))
        if n in p["steps"]:
            assert rel_err(Q, d[f"Q{n}"]) <= 1e-12
            assert rel_err(G, d[f"G{n}"]) <= 1e-10


def test_oracle_kernel_contract_matches_reference():
    """NumPy restatement of the 10-kernel contract vs the reference's
    compiled kernels (same fields as pkg/tests/test_kernels.py)."""
    from oracle import oracle as O
    k = np.load(GOLDEN / "kernels.npz")
    v1, v2 = k["v1"], k["v2"]
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    M = O.k_maxwellian_field_2d(k["rho"], k["u1"], k["u2"], k["T"], v1, v2)
    assert rel_err(M, k["maxwellian"]) <= 1e-12
    args = (k["rho"], k["u1"], k["u2"], k["T"], v1, v2)
    assert rel_err(O.k_project_field_2d(k["G"], M, *args, dv), k["project"]) <= 1e-12
    assert rel_err(O.k_transport_stage_2d(k["Gx"], M, *args, 0.02, 0.003, 0), k["transport0"]) <= 1e-12
    assert rel_err(O.k_transport_stage_2d(k["Gy"], M, *args, 0.02, 0.003, 1), k["transport1"]) <= 1e-12
    gh = O.k_ghat_2d(M, k["rho"], k["u1"], k["u2"], k["T"], k["s11"], k["s12"], k["g1"], k["g2"],
                     k["tau"], v1, v2)
    assert rel_err(gh, k["ghat"]) <= 1e-12
    ga = O.k_add_gaussian_term_2d(k["G"], M, k["rho"], k["u1"], k["u2"], k["m11"], k["m12"],
                                  k["m22"], 0.07, v1, v2)
    assert rel_err(ga, k["gauss"]) <= 1e-12
    assert rel_err(O.k_add_lowrank_4d(k["G"], k["coeffs"], k["shapes"]), k["lowrank"]) <= 1e-12
    assert rel_err(O.k_relax_2d(k["G"], k["Ghat"], k["tau"], 0.004, 0.08), k["relax"]) <= 1e-12
    H = O.k_heat_tensor_2d(k["G"], k["u1"], k["u2"], v1, v2, dv, 0.08)
    for a, b in zip(H, k["heat"]):
        assert rel_err(a, b) <= 1e-12
    assert rel_err(O.k_upwind_z_1d(k["G1x"], k["v"], 0.05), k["upwind1d"]) <= 1e-12
    v40 = k["v40"]
    assert rel_err(O.k_project_field_1d(k["F1"], k["M1"], k["rho1"], k["uu"], k["T1"], v40,
                                        v40[1] - v40[0]), k["project1d"]) <= 1e-12


@pytest.mark.parametrize("case", ["density", "pressure_spd", "pressure_t11", "density_and_spd"])
def test_oracle_reports_reference_error_cell(oracle, case):
    from types import SimpleNamespace as NS
    want = golden_index()["errors"][case]
    Q = np.load(GOLDEN / f"err_{case}_Q.npy")
    mesh = NS(space=(NS(min=0.0, max=1.0, n=6), NS(min=0.0, max=1.0, n=5)),
              velocity=(NS(min=-5.0, max=5.0, n=6), NS(min=-5.0, max=5.0, n=6)))
    bc = NS(left="periodic", right="periodic", bottom="periodic", top="periodic")
    model = NS(kind="esbgk_2d", nu=-0.5, value=1.0)
    prob = oracle.Problem2D(mesh, bc, 0.1, model)
    with pytest.raises(oracle.OracleStateError) as ei:
        oracle.step_2d_arrays(prob, Q, np.zeros((6, 5, 6, 6)), 1e-3)
    assert list(ei.value.cell) == want["cell"]
    assert ei.value.value == pytest.approx(want["value"], rel=1e-14)


# -- manufactured-solution regression pins (reference pkg/tests/test_cases.py:97-107)

def mms_psi(t, x, y):
    return 2.0 + np.sin(2.0 * np.pi * (x - t)) * np.cos(2.0 * np.pi * (y - t))


def mms_psi_derivs(t, x, y):
    a = 2.0 * np.pi * (x - t)
    b = 2.0 * np.pi * (y - t)
    return (-2.0 * np.pi * np.cos(a + b), 2.0 * np.pi * np.cos(a) * np.cos(b),
            -2.0 * np.pi * np.sin(a) * np.sin(b))


def mms_chi(v1, v2):
    return v1 ** 3 - 3.0 * v1 ** 2 * v2 - 3.0 * v1 * v2 ** 2 + v2 ** 3


def mms_problem(n, eps=0.08):
    """The reference's 2D manufactured solution (mms.py:115-179, restated):
    f = e^{-|v|^2} psi (1 + eps chi), rho = pi psi, u = 0, P = pi psi / 2."""
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, PERIODIC,
                                       PhaseMesh, cell_centers, conserved_2d)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, n), Axis(0.0, 1.0, n)),
                     velocity=(Axis(-5.0, 5.0, n), Axis(-5.0, 5.0, n)))
    bc = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
    model = CollisionModel("bgk_2d", nu=0.0)
    x = cell_centers(mesh.space[0])
    y = cell_centers(mesh.space[1])
    v1 = cell_centers(mesh.velocity[0])
    v2 = cell_centers(mesh.velocity[1])
    vel = np.exp(-(v1[:, None] ** 2 + v2[None, :] ** 2)) * mms_chi(v1[:, None], v2[None, :])

    def exact(t):
        psi = mms_psi(t, x[:, None], y[None, :])
        z = np.zeros_like(psi)
        Q = conserved_2d(np.pi * psi, z, z, 0.5 * np.ones_like(psi), z, 0.5 * np.ones_like(psi))
        return Q, psi[:, :, None, None] * vel[None, None]

    def micro_source(t, xx, yy, vv1, vv2):
        X, Y = xx[:, None], yy[None, :]
        al, be, ga = mms_psi_derivs(t, X, Y)
        psi = mms_psi(t, X, Y)
        tau = model.tau(np.pi * psi, 0.5)
        coeffs = np.stack([eps * al + tau * psi, eps * be, eps * ga])
        shapes = np.stack([vel, vel * vv1[:, None], vel * vv2[None, :]])
        return np.ascontiguousarray(coeffs), np.ascontiguousarray(shapes)

    def macro_source(t, xx, yy):
        X, Y = xx[:, None], yy[None, :]
        al, be, ga = mms_psi_derivs(t, X, Y)
        q = 0.75 * eps * np.pi
        return np.stack([np.pi * al, 0.5 * np.pi * be, 0.5 * np.pi * ga,
                         0.5 * np.pi * al + q * (be - ga), -q * (be + ga),
                         0.5 * np.pi * al + q * (ga - be)], axis=-1)

    return mesh, bc, eps, model, exact, micro_source, macro_source


def relative_l2(a, b):
    return math.sqrt(float(np.sum((a - b) ** 2)) / float(np.sum(b * b)))


def test_oracle_reproduces_reference_mms_pin(oracle):
    """mms_run_2d(20): macro 0.030605594996427687, micro 0.031135911051471035
    at rel 1e-12 (reference test_cases.py:104-107, re-measured in index.json)."""
    from paper_2509_21832_b200 import plan_time
    from types import SimpleNamespace as NS
    mesh, bc, eps, model, exact, msrc, qsrc = mms_problem(20)
    plan = plan_time(0.25, 0.926, mesh)
    Q, G = exact(0.0)
    st = NS(t=0.0, Q=Q, G=G)
    for n in range(plan.n_steps):
        _, Qn, Gn, _ = oracle.step_2d(st, mesh, bc, eps, model, plan.dt, micro_source=msrc,
                                      macro_source=qsrc)
        st = NS(t=(n + 1) * plan.dt, Q=Qn, G=Gn)
    Qe, Ge = exact(0.25)
    macro, micro = relative_l2(st.Q, Qe), relative_l2(st.G, Ge)
    pin = golden_index()["mms"]["mms_run_2d_20"]
    assert macro == pytest.approx(0.030605594996427687, rel=1e-12)
    assert micro == pytest.approx(0.031135911051471035, rel=1e-12)
    assert macro == pytest.approx(pin[0], rel=1e-12)


# -- 1D manufactured solution (reference mms.py:1D part, restated) ----------
# f = phi(v) psi(t,x), phi = e^{-(v-1)^2} + 2 e^{-(v+1)^2}, psi = 2 + sin 2pi(x-t);
# exact macro (3 sqrt(pi) psi, -1/3, 25/18); g = (phi - 1.8 e^{-0.04(3v+1)^2}) psi / eps.

MMS1_U, MMS1_T = -1.0 / 3.0, 25.0 / 18.0


def mms1d_problem(n, eps=0.1):
    from paper_2509_21832_b200 import (PERIODIC, Axis, BoundarySpec1D, CollisionModel,
                                       PhaseMesh, cell_centers, conserved_1d)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, n),), velocity=(Axis(-6.5, 6.5, n),))
    bc = BoundarySpec1D(PERIODIC, PERIODIC)
    model = CollisionModel("hard_sphere_1d")
    x = cell_centers(mesh.space[0])
    v = cell_centers(mesh.velocity[0])
    tau = 3.2 * math.sqrt(MMS1_T / (2.0 * math.pi))
    sp = math.sqrt(math.pi)

    def psi(t, xx):
        return 2.0 + np.sin(2.0 * np.pi * (xx - t))

    def phi(vv):
        return np.exp(-(vv - 1.0) ** 2) + 2.0 * np.exp(-(vv + 1.0) ** 2)

    def g_exact(t, xx, vv):
        shape = phi(vv) - 1.8 * np.exp(-0.04 * (3.0 * vv + 1.0) ** 2)
        return psi(t, np.asarray(xx))[:, None] * shape[None, :] / eps

    def h_perp(vv):
        # h - Pi[h] for h = (v-1) phi at the exact state; moments (-4, 5.5, -7) sqrt(pi)
        m0, m1, m2 = -4.0 * sp, 5.5 * sp, -7.0 * sp
        u, T = MMS1_U, MMS1_T
        w = (vv - u) / math.sqrt(T)
        a1 = m0
        a2 = (m1 - u * m0) / math.sqrt(T)
        a3 = math.sqrt(2.0) * ((m2 - 2.0 * u * m1 + u * u * m0) / (2.0 * T) - 0.5 * m0)
        unit = np.exp(-(vv - u) ** 2 / (2.0 * T)) / math.sqrt(2.0 * math.pi * T)
        b3 = math.sqrt(2.0) * (0.5 * w * w - 0.5)
        return (vv - 1.0) * phi(vv) - (a1 + w * a2 + b3 * a3) * unit

    def micro_source(t, xx, vv):
        c = 2.0 * np.pi * np.cos(2.0 * np.pi * (np.asarray(xx) - t))
        return c[:, None] * h_perp(vv)[None, :] + tau * g_exact(t, xx, vv)

    def macro_source(t, xx):
        c = math.pi ** 1.5 * np.cos(2.0 * np.pi * (np.asarray(xx) - t))
        return c[:, None] * np.array([-8.0, 11.0, -7.0])

    def exact(t):
        rho = 3.0 * sp * psi(t, x)
        Q = conserved_1d(rho, np.full_like(rho, MMS1_U), np.full_like(rho, MMS1_T))
        return Q, g_exact(t, x, v)

    return mesh, bc, eps, model, exact, micro_source, macro_source


def test_oracle_reproduces_reference_mms1d_pin(oracle):
    """mms_run_1d(10): macro 0.06653393519741775, micro 0.09812773373649085
    at rel 1e-12 (reference test_cases.py:98-102)."""
    from paper_2509_21832_b200 import cell_centers, plan_time
    mesh, bc, eps, model, exact, msrc, qsrc = mms1d_problem(10)
    plan = plan_time(0.9351, 0.95, mesh)
    prob = oracle.Problem1D(mesh, bc, eps, model)
    x = cell_centers(mesh.space[0])
    Q, G = exact(0.0)
    for n in range(plan.n_steps):
        t = n * plan.dt
        Q, G, _ = oracle.step_1d_arrays(prob, Q, G, plan.dt, src=msrc(t, x, prob.v),
                                        qsrc=qsrc(t, x))
    Qe, Ge = exact(0.9351)
    pin = golden_index()["mms"]["mms_run_1d_10"]
    assert relative_l2(Q, Qe) == pytest.approx(pin[0], rel=1e-12)
    assert relative_l2(G, Ge) == pytest.approx(pin[1], rel=1e-12)

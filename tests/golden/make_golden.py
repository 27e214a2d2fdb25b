"""Generate the golden fixtures by running the REFERENCE solver itself.

Run in the build container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py [--ref /root/reference/pkg]

The reference package is copied to a scratch directory, its Cython kernel
extension is built there (``setup.py build_ext --inplace``), and it is
imported with ``MICROMACRO_BACKEND=compiled``.  Each case drives the
reference's public API -- ``PhaseMesh``/``Axis``, ``BoundarySpec2D``,
``CollisionModel``, ``conserved_2d``, ``State2D``/``step_2d`` (and the 1D
twins) -- exactly as the reference's own tests do (e.g.
pkg/tests/test_parallel.py:26-44), and stores inputs and outputs as
``.npz`` fixtures next to this script.  Nothing here is copied from the
reference; only its outputs are recorded.
"""

from __future__ import annotations

import argparse
import importlib
import json
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def load_reference(ref_pkg: Path):
    work = Path(tempfile.mkdtemp(prefix="mm_ref_"))
    dst = work / "pkg"
    shutil.copytree(ref_pkg, dst, ignore=shutil.ignore_patterns("build", "*.so", "*.c"))
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst,
                   check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    os.environ["MICROMACRO_BACKEND"] = "compiled"
    sys.path.insert(0, str(dst / "src"))
    mm = importlib.import_module("micromacro")
    K = importlib.import_module("micromacro._kernels")
    assert K.backend_name == "compiled", K.backend_name
    return work


def _face_json(f, mm_boundary):
    if isinstance(f, mm_boundary.WallSpec):
        return {"wall": [f.temperature, f.velocity]}
    return f


def cases_2d():
    """(name, params) for every 2D golden case."""
    return [
        # C2-like smooth periodic wave, anisotropic tensor so the ES-BGK cross
        # term is live, nonzero micro field
        ("wave_periodic", dict(nx=12, ny=12, vx=(-7.0, 7.0, 8), vy=(-7.0, 7.0, 8),
                               faces=("periodic",) * 4, kind="esbgk_2d", nu=-0.5,
                               eps=0.1, ic="wave", gscale=0.01, steps=(1, 10, 100))),
        # C3-like four-quadrant Riemann, all faces extrapolate, nx != ny,
        # non-square velocity grid
        ("riemann_extrap", dict(nx=16, ny=12, vx=(-8.0, 8.0, 8), vy=(-8.0, 8.0, 6),
                                faces=("extrapolate",) * 4, kind="esbgk_2d", nu=-0.5,
                                eps=1e-2, ic="riemann", gscale=0.0, steps=(1, 10, 100))),
        ("riemann_extrap_eps1e-3", dict(nx=12, ny=12, vx=(-8.0, 8.0, 8), vy=(-8.0, 8.0, 8),
                                        faces=("extrapolate",) * 4, kind="esbgk_2d", nu=-0.5,
                                        eps=1e-3, ic="riemann", gscale=0.0, steps=(1, 10))),
        # C4-like closed box with diffuse walls on all faces
        ("box_walls", dict(nx=12, ny=12, vx=(-8.0, 8.0, 8), vy=(-8.0, 8.0, 8),
                           faces=({"wall": [1.0, 0.0]},) * 4, kind="esbgk_2d", nu=-0.5,
                           eps=5e-2, ic="bump", gscale=0.005, steps=(1, 10, 100))),
        # lid-driven cavity (reference default case shape), sliding top lid
        ("cavity_lid", dict(nx=10, ny=10, vx=(-5.0, 5.0, 6), vy=(-5.0, 5.0, 6),
                            faces=({"wall": [1.0, 0.0]}, {"wall": [1.0, 0.0]},
                                   {"wall": [1.0, 0.0]}, {"wall": [1.0, 0.16]}),
                            kind="esbgk_2d", nu=-1.0, eps=0.08, ic="smooth", gscale=0.01,
                            steps=(1, 10))),
        # mixed faces, odd velocity counts (V = 63), BGK nu = 0
        ("mixed_oddv", dict(nx=8, ny=10, vx=(-5.0, 5.0, 7), vy=(-6.0, 6.0, 9),
                            faces=("extrapolate", "extrapolate", "periodic", "periodic"),
                            kind="bgk_2d", nu=0.0, eps=0.3, ic="smooth", gscale=0.01,
                            steps=(1, 10))),
        # periodic x, hot sliding wall at the bottom, extrapolate top,
        # constant tau
        ("mixed_walls", dict(nx=10, ny=8, vx=(-6.0, 6.0, 8), vy=(-6.0, 6.0, 8),
                             faces=("periodic", "periodic", {"wall": [1.2, 0.1]}, "extrapolate"),
                             kind="constant", nu=-0.3, eps=0.05, ic="smooth", gscale=0.01,
                             steps=(1, 10))),
        # asymptotic limit with an isotropic tensor: the eps < 1e-10 guard
        # skips the Gaussian term (micro2d.py:96)
        ("ap_isotropic", dict(nx=8, ny=8, vx=(-6.0, 6.0, 8), vy=(-6.0, 6.0, 8),
                              faces=("periodic",) * 4, kind="esbgk_2d", nu=-1.0,
                              eps=1e-14, ic="iso", gscale=0.0, steps=(1,))),
        # benchmark velocity grid (32 x 32 = 1024 nodes per cell)
        ("wave_v1024", dict(nx=6, ny=6, vx=(-7.0, 7.0, 32), vy=(-7.0, 7.0, 32),
                            faces=("periodic",) * 4, kind="esbgk_2d", nu=-0.5,
                            eps=0.1, ic="wave", gscale=0.01, steps=(1, 3))),
        ("box_v1024", dict(nx=6, ny=6, vx=(-8.0, 8.0, 32), vy=(-8.0, 8.0, 32),
                           faces=({"wall": [1.0, 0.0]},) * 4, kind="esbgk_2d", nu=-0.5,
                           eps=5e-2, ic="bump", gscale=0.005, steps=(1, 3))),
        # (round 2) the eps < 1e-10 isotropy guard (micro2d.py:96) on the
        # benchmark velocity grid, i.e. on the specialised 32 x 32 kernel:
        # isotropic tensor -> the Gaussian term is skipped ...
        ("iso_v1024_eps1e-12", dict(nx=6, ny=6, vx=(-7.0, 7.0, 32), vy=(-7.0, 7.0, 32),
                                    faces=("periodic",) * 4, kind="esbgk_2d", nu=-0.5,
                                    eps=1e-12, ic="iso", gscale=0.0, steps=(1,))),
        # (only one step: after it the physical anisotropy is O(eps) = 1e-12,
        # at the guard's own 1e-13 max T threshold, so whether later steps
        # take the Gaussian term is decided by roundoff)
        # ... anisotropic tensor -> the guard does not fire, (G - M)/eps is live
        ("wave_v1024_eps1e-12", dict(nx=6, ny=6, vx=(-7.0, 7.0, 32), vy=(-7.0, 7.0, 32),
                                     faces=("periodic",) * 4, kind="esbgk_2d", nu=-0.5,
                                     eps=1e-12, ic="wave", gscale=0.0, steps=(1,))),
        # (one step as well: the macro relaxation at eps = 1e-12 makes the
        # tensor isotropic to ~1e-13, the guard's knife edge, from step 2 on)
    ]


def initial_state(p, mm, rng):
    from micromacro.gas_state import conserved_2d
    from micromacro.mesh import cell_centers
    nx, ny = p["nx"], p["ny"]
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y, indexing="ij")
    ic = p["ic"]
    if ic == "wave":
        rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)
        u1 = 0.5 + 0.05 * np.cos(2 * np.pi * Y)
        u2 = 0.5 - 0.04 * np.sin(2 * np.pi * X)
        t11 = 1.0 + 0.1 * np.cos(2 * np.pi * X)
        t22 = 1.0 - 0.05 * np.sin(2 * np.pi * Y)
        t12 = 0.05 * np.sin(2 * np.pi * (X + Y))
    elif ic == "riemann":
        north = Y >= 0.5
        east = X >= 0.5
        rho = np.where(north, np.where(east, 1.0, 0.5), np.where(east, 0.5, 0.25))
        u1 = np.where(north, np.where(east, 0.0, 0.5), np.where(east, 0.0, 0.5))
        u2 = np.where(north, np.where(east, 0.0, 0.0), np.where(east, 0.5, 0.5))
        T = np.where(north, np.where(east, 1.0, 0.8), np.where(east, 0.8, 0.6))
        t11, t22, t12 = T, T, np.zeros_like(T)
    elif ic == "bump":
        rho = 1.0 + 0.5 * np.exp(-((X - 0.3) ** 2 + (Y - 0.6) ** 2) / 0.01)
        u1 = np.zeros_like(X)
        u2 = np.zeros_like(X)
        t11 = np.ones_like(X)
        t22 = np.ones_like(X)
        t12 = np.zeros_like(X)
    elif ic == "iso":
        rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)
        u1 = 0.1 * np.cos(2 * np.pi * Y)
        u2 = -0.1 * np.sin(2 * np.pi * X)
        T = 1.0 + 0.1 * np.cos(2 * np.pi * X)
        t11, t22, t12 = T, T, np.zeros_like(T)
    else:  # smooth
        rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)
        u1 = 0.02 * np.cos(2 * np.pi * Y)
        u2 = -0.03 * np.sin(2 * np.pi * X)
        t11 = 1.0 + 0.1 * np.cos(2 * np.pi * X)
        t22 = 1.0 + 0.08 * np.sin(2 * np.pi * Y)
        t12 = 0.03 * np.cos(2 * np.pi * (X - Y))
    Q = conserved_2d(rho, u1, u2, t11, t12, t22)
    nv1, nv2 = p["vx"][2], p["vy"][2]
    G = p["gscale"] * rng.standard_normal((nx, ny, nv1, nv2))
    return Q, G


def make_2d(outdir: Path, index):
    from micromacro.boundary import (EXTRAPOLATE, PERIODIC, BoundarySpec2D, WallSpec)
    from micromacro.gas_state import CollisionModel
    from micromacro.macro2d import heat_flux_tensor_2d
    from micromacro.mesh import Axis, PhaseMesh, cell_centers
    from micromacro.runner.loop import State2D, step_2d
    from micromacro.gas_state import primitives_2d

    def face(f):
        if isinstance(f, dict):
            return WallSpec(temperature=f["wall"][0], velocity=f["wall"][1])
        return {"periodic": PERIODIC, "extrapolate": EXTRAPOLATE}[f]

    for seed, (name, p) in enumerate(cases_2d()):
        rng = np.random.default_rng(1000 + seed)
        mesh = PhaseMesh(space=(Axis(0.0, 1.0, p["nx"]), Axis(0.0, 1.0, p["ny"])),
                         velocity=(Axis(*p["vx"]), Axis(*p["vy"])))
        bc = BoundarySpec2D(*(face(f) for f in p["faces"]))
        model = CollisionModel(p["kind"], nu=p["nu"], value=0.7)
        Q0, G0 = initial_state(p, None, rng)
        vmax = max(abs(p["vx"][0]), abs(p["vx"][1]), abs(p["vy"][0]), abs(p["vy"][1]))
        dt = 0.4 * min(1.0 / p["nx"], 1.0 / p["ny"]) / vmax
        state = State2D(t=0.0, Q=np.array(Q0), G=np.array(G0))
        out = dict(Q0=Q0, G0=G0, dt=dt)
        v1 = cell_centers(mesh.velocity[0])
        v2 = cell_centers(mesh.velocity[1])
        last = max(p["steps"])
        for n in range(1, last + 1):
            _, u1, u2, _, _, _ = primitives_2d(state.Q)
            new = step_2d(state, mesh, bc, p["eps"], model, dt)
            if n in p["steps"]:
                Hstep = np.array(heat_flux_tensor_2d(new.G, u1, u2, v1, v2, p["eps"]))
                _, u1n, u2n, _, _, _ = primitives_2d(new.Q)
                Hframe = np.array(heat_flux_tensor_2d(new.G, u1n, u2n, v1, v2, p["eps"]))
                out[f"Q{n}"] = new.Q
                out[f"G{n}"] = new.G
                out[f"Hstep{n}"] = Hstep
                out[f"Hframe{n}"] = Hframe
            state = new
        np.savez_compressed(outdir / f"step2d_{name}.npz", **out)
        index[f"step2d_{name}"] = {**{k: v for k, v in p.items()}, "tau_value": 0.7,
                                   "dt": dt}
        print("wrote", name)


def make_configs(outdir: Path, index, n=12):
    """The BASELINE configurations exactly as bench.py builds them
    (bench.workload_spec + bench.initial_prims: same generators, velocity
    grids, faces, eps, nu, dt rule), at n x n cells so the reference runs
    100 steps in seconds.  Stores Q and both heat tensors after 1, 10 and 100
    steps (G after 100 steps for the wall box and the C5 generator)."""
    sys.path.insert(0, str(HERE.parents[1]))
    import bench
    from micromacro.boundary import EXTRAPOLATE, PERIODIC, BoundarySpec2D, WallSpec
    from micromacro.gas_state import CollisionModel, conserved_2d, primitives_2d
    from micromacro.macro2d import heat_flux_tensor_2d
    from micromacro.mesh import Axis, PhaseMesh, cell_centers
    from micromacro.runner.loop import State2D, step_2d
    cases = [("c2", None), ("c3", 1e-3), ("c3", 1e-2), ("c3", 1e-1), ("c4", None), ("c5", None)]
    for name, eps in cases:
        spec = bench.workload_spec(name, n=n, eps=eps)
        lo, hi, nv = spec["vel"]
        mesh = PhaseMesh(space=(Axis(0.0, spec["Lx"], n), Axis(0.0, spec["Ly"], n)),
                         velocity=(Axis(lo, hi, nv), Axis(lo, hi, nv)))
        if spec["faces"] == "periodic":
            bc = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
        elif spec["faces"] == "extrapolate":
            bc = BoundarySpec2D(EXTRAPOLATE, EXTRAPOLATE, EXTRAPOLATE, EXTRAPOLATE)
        else:
            w = WallSpec(temperature=1.0, velocity=0.0)
            bc = BoundarySpec2D(w, w, w, w)
        model = CollisionModel(spec["kind"], nu=spec["nu"])
        rho, u1, u2, T = bench.initial_prims(spec, 0, n, 0, n)
        Q0 = conserved_2d(rho, u1, u2, T, 0 * T, T)
        st = State2D(t=0.0, Q=np.array(Q0), G=np.zeros((n, n, nv, nv)))
        v1 = cell_centers(mesh.velocity[0])
        v2 = cell_centers(mesh.velocity[1])
        out = dict(Q0=Q0, dt=spec["dt"])
        for k in range(1, 101):
            _, u1n, u2n, _, _, _ = primitives_2d(st.Q)
            new = step_2d(st, mesh, bc, spec["eps"], model, spec["dt"])
            if k in (1, 10, 100):
                out[f"Q{k}"] = new.Q
                out[f"Hstep{k}"] = np.array(heat_flux_tensor_2d(new.G, u1n, u2n, v1, v2, spec["eps"]))
                _, a1, a2, _, _, _ = primitives_2d(new.Q)
                out[f"Hframe{k}"] = np.array(heat_flux_tensor_2d(new.G, a1, a2, v1, v2, spec["eps"]))
                if k == 100 and name in ("c4", "c5"):
                    out["G100"] = new.G
            st = new
        tag = f"cfg_{name}" + (f"_eps{eps:g}" if eps is not None else "") + f"_n{n}"
        np.savez_compressed(outdir / f"{tag}.npz", **out)
        index[tag] = {"config": name, "n": n, "eps": spec["eps"], "dt": spec["dt"],
                      "faces": spec["faces"], "seed": spec["seed"], "steps": [1, 10, 100],
                      "generator": "bench.workload_spec / bench.initial_prims"}
        print("wrote", tag)


def make_errors(outdir: Path, index):
    """InvalidStateError cases: the reference's cell and value."""
    from micromacro.boundary import PERIODIC, BoundarySpec2D
    from micromacro.errors import InvalidStateError
    from micromacro.gas_state import CollisionModel, conserved_2d
    from micromacro.mesh import Axis, PhaseMesh
    from micromacro.runner.loop import State2D, step_2d
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, 6), Axis(0.0, 1.0, 5)),
                     velocity=(Axis(-5.0, 5.0, 6), Axis(-5.0, 5.0, 6)))
    bc = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
    model = CollisionModel("esbgk_2d", nu=-0.5)
    results = {}
    base = conserved_2d(np.ones((6, 5)), 0.1, -0.1, 1.0, 0.0, 1.0)
    variants = {}
    q = base.copy(); q[3, 2, 0] = -0.5; q[4, 1, 0] = -1.0; variants["density"] = q
    q = base.copy(); q[2, 4, 4] = 5.0; variants["pressure_spd"] = q   # |T12| > sqrt(T11 T22)
    q = base.copy(); q[1, 3, 3] = 0.005; variants["pressure_t11"] = q
    # (round 2) several failing cells of different checks: the reference
    # checks density over the whole field before the tensor, so the density
    # cell is raised although an SPD failure sits at an earlier cell
    q = base.copy(); q[0, 1, 4] = 5.0; q[4, 3, 0] = -0.2; q[5, 4, 0] = -0.1
    variants["density_and_spd"] = q
    for name, Q in variants.items():
        try:
            step_2d(State2D(0.0, Q, np.zeros((6, 5, 6, 6))), mesh, bc, 0.1, model, 1e-3)
            results[name] = None
        except InvalidStateError as e:
            results[name] = {"message": str(e), "cell": [int(c) for c in e.cell],
                             "value": float(e.value)}
        np.save(outdir / f"err_{name}_Q.npy", Q)
    index["errors"] = results
    print("wrote errors", results)


def make_mms(outdir: Path, index):
    """The reference's own frozen MMS regression values
    (pkg/tests/test_cases.py:97-107), re-measured here."""
    from micromacro.runner.cases import mms_run_1d, mms_run_2d
    m1 = mms_run_1d(10)
    m2 = mms_run_2d(20)
    index["mms"] = {"mms_run_1d_10": list(m1), "mms_run_2d_20": list(m2)}
    print("mms", m1, m2)


def make_1d(outdir: Path, index):
    from micromacro.boundary import (EXTRAPOLATE, PERIODIC, BoundarySpec1D, WallSpec)
    from micromacro.gas_state import CollisionModel, conserved_1d
    from micromacro.mesh import Axis, PhaseMesh, plan_time
    from micromacro.runner.loop import State1D, step_1d
    cases = [
        ("sod", dict(nx=64, v=(-8.0, 8.0, 32), faces=("extrapolate", "extrapolate"),
                     kind="hard_sphere_1d", eps=1e-2, ic="sod", steps=(1, 20))),
        ("heat_walls", dict(nx=32, v=(-6.0, 6.0, 24), faces=({"wall": 1.0}, {"wall": 1.2}),
                            kind="pressure_1d", eps=1e-2, ic="uniform", steps=(1, 20))),
        ("periodic", dict(nx=32, v=(-6.5, 6.5, 40), faces=("periodic", "periodic"),
                          kind="hard_sphere_1d", eps=0.1, ic="wave", steps=(1, 20))),
    ]

    def face(f):
        if isinstance(f, dict):
            return WallSpec(temperature=f["wall"])
        return {"periodic": PERIODIC, "extrapolate": EXTRAPOLATE}[f]

    for seed, (name, p) in enumerate(cases):
        rng = np.random.default_rng(2000 + seed)
        nx = p["nx"]
        mesh = PhaseMesh(space=(Axis(0.0, 1.0, nx),), velocity=(Axis(*p["v"]),))
        bc = BoundarySpec1D(*(face(f) for f in p["faces"]))
        model = CollisionModel(p["kind"])
        x = (np.arange(nx) + 0.5) / nx
        if p["ic"] == "sod":
            Q0 = conserved_1d(np.where(x < 0.5, 1.0, 0.125), np.zeros(nx),
                              np.where(x < 0.5, 1.0, 0.8))
            G0 = np.zeros((nx, p["v"][2]))
        elif p["ic"] == "uniform":
            Q0 = conserved_1d(np.ones(nx), np.zeros(nx), 1.0 + 0.1 * x)
            G0 = np.zeros((nx, p["v"][2]))
        else:
            Q0 = conserved_1d(1.0 + 0.3 * np.sin(2 * np.pi * x), 0.2 + 0.1 * np.cos(2 * np.pi * x),
                              1.0 + 0.2 * np.sin(4 * np.pi * x))
            G0 = 0.01 * rng.standard_normal((nx, p["v"][2]))
        dt = 0.4 * (1.0 / nx) / max(abs(p["v"][0]), abs(p["v"][1]))
        st = State1D(0.0, np.array(Q0), np.array(G0))
        out = dict(Q0=Q0, G0=G0, dt=dt)
        for n in range(1, max(p["steps"]) + 1):
            st = step_1d(st, mesh, bc, p["eps"], model, dt)
            if n in p["steps"]:
                out[f"Q{n}"] = st.Q
                out[f"G{n}"] = st.G
        np.savez_compressed(outdir / f"step1d_{name}.npz", **out)
        index[f"step1d_{name}"] = {**p, "dt": dt}
        print("wrote 1d", name)


def make_kernels(outdir: Path, index):
    """Per-kernel outputs of the reference's compiled plugin API on the
    field shapes its own cross-backend test uses (test_kernels.py:13-36)."""
    from micromacro._kernels import _core as K
    rng = np.random.default_rng(123)
    NX, NY, NV1, NV2 = 6, 5, 12, 10
    v1 = np.linspace(-5.7, 5.7, NV1)
    v2 = np.linspace(-6.1, 6.1, NV2)
    rho = rng.uniform(0.5, 1.5, (NX, NY))
    u1 = rng.uniform(-0.5, 0.5, (NX, NY))
    u2 = rng.uniform(-0.5, 0.5, (NX, NY))
    T = rng.uniform(0.7, 1.4, (NX, NY))
    tau = rng.uniform(0.3, 1.2, (NX, NY))
    G = rng.standard_normal((NX, NY, NV1, NV2))
    Gx = rng.standard_normal((NX + 2, NY, NV1, NV2))
    Gy = rng.standard_normal((NX, NY + 2, NV1, NV2))
    s11, s12, g1, g2 = (rng.standard_normal((NX, NY)) for _ in range(4))
    m11 = rng.uniform(0.8, 1.2, (NX, NY))
    m12 = rng.uniform(-0.2, 0.2, (NX, NY))
    m22 = rng.uniform(0.8, 1.2, (NX, NY))
    coeffs = rng.standard_normal((3, NX, NY))
    shapes = rng.standard_normal((3, NV1, NV2))
    Ghat = rng.standard_normal((NX, NY, NV1, NV2))
    nv = 16
    v = np.linspace(-6.5, 6.5, nv)
    G1x = rng.standard_normal((NX + 2, nv))
    nv40 = 40
    v40 = np.linspace(-6.5, 6.5, nv40)
    rho1 = rng.uniform(0.5, 1.5, NX)
    uu = rng.uniform(-0.5, 0.5, NX)
    T1 = rng.uniform(0.7, 1.3, NX)
    M1 = rho1[:, None] / np.sqrt(2 * np.pi * T1[:, None]) * np.exp(-(v40[None, :] - uu[:, None]) ** 2 / (2 * T1[:, None]))
    F1 = rng.standard_normal((NX, nv40))
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    c = np.ascontiguousarray
    M = K.maxwellian_field_2d(rho, u1, u2, T, v1, v2)
    out = dict(v1=v1, v2=v2, rho=rho, u1=u1, u2=u2, T=T, tau=tau, G=G, Gx=Gx, Gy=Gy,
               s11=s11, s12=s12, g1=g1, g2=g2, m11=m11, m12=m12, m22=m22,
               coeffs=coeffs, shapes=shapes, Ghat=Ghat, v=v, G1x=G1x, v40=v40,
               rho1=rho1, uu=uu, T1=T1, M1=M1, F1=F1)
    out["maxwellian"] = M
    out["project"] = K.project_field_2d(G, M, rho, u1, u2, T, v1, v2, dv)
    out["transport0"] = K.transport_stage_2d(Gx, M, rho, u1, u2, T, v1, v2, 0.02, 0.003, 0)
    out["transport1"] = K.transport_stage_2d(Gy, M, rho, u1, u2, T, v1, v2, 0.02, 0.003, 1)
    out["ghat"] = K.ghat_2d(M, rho, u1, u2, T, s11, s12, g1, g2, tau, v1, v2)
    a = np.array(G, copy=True)
    K.add_gaussian_term_2d(a, M, rho, u1, u2, m11, m12, m22, 0.07, v1, v2)
    out["gauss"] = a
    a = np.array(G, copy=True)
    K.add_lowrank_4d(a, c(coeffs), c(shapes))
    out["lowrank"] = a
    out["relax"] = K.relax_2d(G, Ghat, tau, 0.004, 0.08)
    out["heat"] = np.array(K.heat_tensor_2d(G, u1, u2, v1, v2, dv, 0.08))
    out["upwind1d"] = K.upwind_z_1d(c(G1x), v, 0.05)
    out["project1d"] = K.project_field_1d(c(F1), c(M1), rho1, uu, T1, v40, v40[1] - v40[0])
    np.savez_compressed(outdir / "kernels.npz", **out)
    index["kernels"] = {"NX": NX, "NY": NY, "NV1": NV1, "NV2": NV2}
    print("wrote kernels")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    work = load_reference(Path(args.ref))
    index = {"generator": "tests/golden/make_golden.py",
             "reference_backend": "compiled",
             "numpy": np.__version__}
    try:
        import scipy
        index["scipy"] = scipy.__version__
        make_kernels(HERE, index)
        make_2d(HERE, index)
        make_configs(HERE, index)
        make_1d(HERE, index)
        make_errors(HERE, index)
        make_mms(HERE, index)
    finally:
        shutil.rmtree(work, ignore_errors=True)
    with open(HERE / "index.json", "w") as fh:
        json.dump(index, fh, indent=1, default=str)


if __name__ == "__main__":
    main()

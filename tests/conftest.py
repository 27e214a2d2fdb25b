"""Shared fixtures.  ``-m gpu`` tests need a B200 (they run the CUDA path
through the C ABI); everything else runs on the CPU (oracle vs reference
goldens, host logic, ABI exports, gloo multi-process logic)."""

import json
import sys
from pathlib import Path
from types import SimpleNamespace as NS

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libmm2d.so")


def golden_index():
    with open(GOLDEN / "index.json") as fh:
        return json.load(fh)


def golden_cases(prefix):
    return sorted(k for k in golden_index() if k.startswith(prefix))


def problem_from_golden(name):
    """(mesh, bc, eps, model, params) built with this repo's drop-in API."""
    from paper_2509_21832_b200 import (Axis, BoundarySpec2D, CollisionModel, EXTRAPOLATE,
                                       PERIODIC, PhaseMesh, WallSpec)
    p = golden_index()[name]

    def face(f):
        if isinstance(f, dict):
            return WallSpec(temperature=f["wall"][0], velocity=f["wall"][1])
        return {"periodic": PERIODIC, "extrapolate": EXTRAPOLATE}[f]

    mesh = PhaseMesh(space=(Axis(0.0, 1.0, p["nx"]), Axis(0.0, 1.0, p["ny"])),
                     velocity=(Axis(*p["vx"]), Axis(*p["vy"])))
    bc = BoundarySpec2D(*(face(f) for f in p["faces"]))
    model = CollisionModel(p["kind"], nu=p["nu"], value=p.get("tau_value", 0.7))
    return mesh, bc, p["eps"], model, p


def problem1d_from_golden(name):
    """1D (mesh, bc, eps, model, params) built with this repo's drop-in API."""
    from paper_2509_21832_b200 import (Axis, BoundarySpec1D, CollisionModel, EXTRAPOLATE,
                                       PERIODIC, PhaseMesh, WallSpec)
    p = golden_index()[name]

    def face(f):
        if isinstance(f, dict):
            return WallSpec(temperature=f["wall"])
        return {"periodic": PERIODIC, "extrapolate": EXTRAPOLATE}[f]

    mesh = PhaseMesh(space=(Axis(0.0, 1.0, p["nx"]),), velocity=(Axis(*p["v"]),))
    bc = BoundarySpec1D(*(face(f) for f in p["faces"]))
    model = CollisionModel(p["kind"])
    return mesh, bc, p["eps"], model, p


def q1_rel_err(Q, Qref):
    """1D moments: max over (rho, rho u, E) of the rel L-inf error; momentum
    is floored at max rho * sqrt(max T)."""
    rho = Qref[:, 0]
    T = 2.0 * Qref[:, 2] / rho - (Qref[:, 1] / rho) ** 2
    s = [float(np.max(np.abs(Qref[:, c]))) for c in range(3)]
    s[1] = max(s[1], float(np.max(rho)) * float(np.sqrt(np.max(T))))
    return max(float(np.max(np.abs(Q[:, c] - Qref[:, c]))) / s[c] for c in range(3))


def q_scales(Qref):
    """Per-component error scales for moment comparisons (SURVEY 8c floors:
    momentum uses max rho * sqrt(max T); E12 uses the diagonal maxima)."""
    rho = Qref[..., 0]
    u1 = Qref[..., 1] / rho
    u2 = Qref[..., 2] / rho
    T = 0.5 * (Qref[..., 3] / rho - u1 * u1 + Qref[..., 5] / rho - u2 * u2)
    mom_floor = float(np.max(rho)) * float(np.sqrt(np.max(T)))
    diag = max(float(np.max(np.abs(Qref[..., 3]))), float(np.max(np.abs(Qref[..., 5]))))
    s = [float(np.max(np.abs(Qref[..., c]))) for c in range(6)]
    s[1] = max(s[1], mom_floor)
    s[2] = max(s[2], mom_floor)
    s[4] = max(s[4], diag)
    return np.array(s)


def q_rel_err(Q, Qref):
    """max over components of rel L-inf error with the floors above."""
    sc = q_scales(Qref)
    return max(float(np.max(np.abs(Q[..., c] - Qref[..., c]))) / sc[c] for c in range(6))


def prims(Q):
    """rho, u1, u2, T11, T12, T22, T, p of (..., 6) moments
    (gas_state.py:93-108: u = m / rho, T_ab = E_ab / rho - u_a u_b,
    T = (T11 + T22) / 2, p = rho T)."""
    rho = Q[..., 0]
    u1 = Q[..., 1] / rho
    u2 = Q[..., 2] / rho
    t11 = Q[..., 3] / rho - u1 * u1
    t12 = Q[..., 4] / rho - u1 * u2
    t22 = Q[..., 5] / rho - u2 * u2
    T = 0.5 * (t11 + t22)
    return [rho, u1, u2, t11, t12, t22, T, rho * T]


PRIM_NAMES = ("rho", "u1", "u2", "T11", "T12", "T22", "T", "p")


def prim_rel_errs(Q, Qref):
    """Rel L-inf error of every primitive moment, with the SURVEY 8c floors:
    velocities use sqrt(max T), T12 the diagonal maxima."""
    a, b = prims(Q), prims(Qref)
    scale = [float(np.max(np.abs(x))) for x in b]
    sqrtT = float(np.sqrt(np.max(b[6])))
    scale[1] = max(scale[1], sqrtT)
    scale[2] = max(scale[2], sqrtT)
    scale[4] = max(scale[4], scale[3], scale[5])
    return {n: float(np.max(np.abs(x - y))) / s for n, x, y, s in zip(PRIM_NAMES, a, b, scale)}


def prim_rel_err(Q, Qref):
    return max(prim_rel_errs(Q, Qref).values())


def h_rel_err(H, Href, Qref, eps):
    """Heat tensor error relative to max(max |Href|, 1e-4 eps rho T^1.5):
    the floor keeps roundoff-level heat tensors (e.g. C2's first step, where
    the micro field is pure roundoff) from being graded as signal."""
    p = prims(Qref)
    floor = 1e-4 * eps * float(np.max(p[0])) * float(np.max(p[6])) ** 1.5
    return float(np.max(np.abs(np.asarray(H) - np.asarray(Href)))) / max(
        float(np.max(np.abs(Href))), floor)


def heat_sum_scale(G, eps, v1, v2):
    """eps dv max_cell sum_n |v|^3 |G_n|: the magnitude of the terms the heat
    tensor sums.  When they cancel to many digits (eps -> 0 with an
    anisotropic tensor: G ~ (Gaussian - M) / eps is huge while its heat
    moment is tiny) a different summation order legitimately differs by
    roundoff of THIS scale, so 1e-5 of it floors heat-tensor comparisons."""
    v1 = np.asarray(v1)
    v2 = np.asarray(v2)
    vmax = max(float(np.max(np.abs(v1))), float(np.max(np.abs(v2))))
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    return eps * dv * vmax ** 3 * float(np.max(np.sum(np.abs(G), axis=(-2, -1))))


def rel_err(a, b, floor=1e-300):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), floor)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O

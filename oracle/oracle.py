"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

The oracle (``mm_oracle.c``) is a plain-C restatement of the reference
solver's timestep (see that file's header for the per-function citations).
This module is imported only by ``tests/``, ``__graft_entry__.smoke()`` and
the CPU-baseline leg of ``bench.py``; the product package never touches it.

Objects describing the problem (mesh, boundary spec, collision model) are
read by duck typing, so both the reference's own ``micromacro`` objects and
this repo's drop-in objects work.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libmm_oracle.so"

FACE_PERIODIC, FACE_EXTRAPOLATE, FACE_WALL, FACE_SPECULAR = 0, 1, 2, 3
TAU_KINDS = {"hard_sphere_1d": 0, "pressure_1d": 1, "esbgk_2d": 2,
             "bgk_2d": 3, "constant": 4}
ERR_MESSAGES = {1: "non-positive density",
                2: "pressure tensor is not positive definite",
                3: "modified temperature tensor is not positive definite",
                4: "non-positive temperature"}

_dp = C.POINTER(C.c_double)


class _Err(C.Structure):
    _fields_ = [("code", C.c_int), ("i", C.c_int), ("j", C.c_int),
                ("value", C.c_double)]


class _Cfg2D(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nv1", C.c_int),
                ("nv2", C.c_int), ("dx", C.c_double), ("dy", C.c_double),
                ("v1", _dp), ("v2", _dp), ("face", C.c_int * 4),
                ("wall_T", C.c_double * 4), ("wall_U", C.c_double * 4),
                ("tau_kind", C.c_int), ("tau_value", C.c_double),
                ("nu", C.c_double), ("eps", C.c_double)]


class _Cfg1D(C.Structure):
    _fields_ = [("nx", C.c_int), ("nv", C.c_int), ("dx", C.c_double),
                ("v", _dp), ("face", C.c_int * 2), ("wall_T", C.c_double * 2),
                ("tau_kind", C.c_int), ("tau_value", C.c_double),
                ("eps", C.c_double)]


class OracleStateError(RuntimeError):
    """The oracle found a non-physical state (mirrors InvalidStateError)."""

    def __init__(self, message, cell, value):
        super().__init__(f"{message} at cell {cell} (value {value})")
        self.cell = cell
        self.value = value


_lib = None


def build():
    """Compile the oracle library (gcc) if it is missing or stale."""
    src = _HERE / "mm_oracle.c"
    if (not _LIB_PATH.exists()
            or _LIB_PATH.stat().st_mtime < src.stat().st_mtime):
        subprocess.run(["make", "-C", str(_HERE)], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(_LIB_PATH))
        _lib.mmo_step_2d.restype = C.c_int
        _lib.mmo_step_1d.restype = C.c_int
        _lib.mmo_num_threads.restype = C.c_int
    return _lib


def set_num_threads(n):
    lib().mmo_set_num_threads(int(n))


def num_threads():
    return int(lib().mmo_num_threads())


def _p(a):
    return a.ctypes.data_as(_dp)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _centers(axis):
    return axis.min + (np.arange(1, axis.n + 1) - 0.5) * ((axis.max - axis.min) / axis.n)


def _face_code(face):
    if isinstance(face, str):
        return {"periodic": FACE_PERIODIC, "extrapolate": FACE_EXTRAPOLATE,
                "specular": FACE_SPECULAR}[face]
    return FACE_WALL


class Problem2D:
    """Flattened description of a 2D step problem (duck-typed inputs)."""

    def __init__(self, mesh, bc, eps, model):
        sx, sy = mesh.space
        vx, vy = mesh.velocity
        self.nx, self.ny, self.nv1, self.nv2 = sx.n, sy.n, vx.n, vy.n
        self.dx = (sx.max - sx.min) / sx.n
        self.dy = (sy.max - sy.min) / sy.n
        self.v1 = _c64(_centers(vx))
        self.v2 = _c64(_centers(vy))
        faces = (bc.left, bc.right, bc.bottom, bc.top)
        self.face = [_face_code(f) for f in faces]
        self.wall_T = [getattr(f, "temperature", 0.0) for f in faces]
        self.wall_U = [getattr(f, "velocity", 0.0) for f in faces]
        self.tau_kind = TAU_KINDS[model.kind]
        self.tau_value = float(getattr(model, "value", 1.0))
        self.nu = float(model.nu)
        self.eps = float(eps)

    def cfg(self):
        c = _Cfg2D()
        c.nx, c.ny, c.nv1, c.nv2 = self.nx, self.ny, self.nv1, self.nv2
        c.dx, c.dy = self.dx, self.dy
        c.v1, c.v2 = _p(self.v1), _p(self.v2)
        for f in range(4):
            c.face[f] = self.face[f]
            c.wall_T[f] = self.wall_T[f]
            c.wall_U[f] = self.wall_U[f]
        c.tau_kind, c.tau_value = self.tau_kind, self.tau_value
        c.nu, c.eps = self.nu, self.eps
        return c


def step_2d_arrays(prob: Problem2D, Q, G, dt, src=None, qsrc=None):
    """One oracle step: returns (Q_new, G_new, H) with H (4, nx, ny) the
    u^n-based heat tensor used inside the step (loop.py:108)."""
    Q = _c64(Q)
    G = _c64(G)
    nx, ny = prob.nx, prob.ny
    Qo = np.empty_like(Q)
    Go = np.empty_like(G)
    H = np.empty((4, nx, ny))
    err = _Err()
    nsrc = 0
    sc = ss = None
    if src is not None:
        coeffs, shapes = src
        sc = _c64(coeffs)
        ss = _c64(shapes)
        nsrc = sc.shape[0]
    qs = _c64(qsrc) if qsrc is not None else None
    cfg = prob.cfg()
    rc = lib().mmo_step_2d(C.byref(cfg), _p(Q), _p(G), C.c_double(dt),
                           C.c_int(nsrc), _p(sc) if sc is not None else None,
                           _p(ss) if ss is not None else None,
                           _p(qs) if qs is not None else None,
                           _p(Qo), _p(Go), _p(H), C.byref(err))
    if rc != 0:
        raise OracleStateError(ERR_MESSAGES.get(err.code, "invalid state"),
                               (err.i, err.j), err.value)
    return Qo, Go, H


def step_2d(state, mesh, bc, eps, model, dt, micro_source=None,
            macro_source=None):
    """Oracle twin of ``micromacro.runner.loop.step_2d`` (loop.py:82-111).

    ``state`` needs ``t``, ``Q`` and ``G``; returns a ``(t, Q, G, H)`` tuple.
    """
    prob = Problem2D(mesh, bc, eps, model)
    src = qsrc = None
    if micro_source is not None or macro_source is not None:
        x = _centers(mesh.space[0])
        y = _centers(mesh.space[1])
        if micro_source is not None:
            src = micro_source(state.t, x, y, prob.v1, prob.v2)
        if macro_source is not None:
            qsrc = macro_source(state.t, x, y)
    Q, G, H = step_2d_arrays(prob, state.Q, state.G, dt, src, qsrc)
    return state.t + dt, Q, G, H


def run_steps_2d(prob: Problem2D, Q, G, dt, n_steps):
    for _ in range(n_steps):
        Q, G, H = step_2d_arrays(prob, Q, G, dt)
    return Q, G, H


def heat_tensor_2d(G, u1, u2, v1, v2, eps):
    """heat_flux_tensor_2d (macro2d.py:23-29) via the oracle kernel."""
    G = _c64(G)
    nx, ny, nv1, nv2 = G.shape
    u1, u2, v1, v2 = (_c64(a) for a in (u1, u2, v1, v2))
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    H = np.empty((4, nx, ny))
    lib().mmo_heat_tensor_2d(nx, ny, nv1, nv2, _p(G), _p(u1), _p(u2), _p(v1),
                             _p(v2), C.c_double(dv), C.c_double(eps), _p(H))
    return H


def primitives_2d(Q):
    """(rho, u1, u2, T11, T12, T22, T) without validation."""
    Q = np.asarray(Q, dtype=float)
    rho = Q[..., 0]
    u1 = Q[..., 1] / rho
    u2 = Q[..., 2] / rho
    t11 = Q[..., 3] / rho - u1 * u1
    t12 = Q[..., 4] / rho - u1 * u2
    t22 = Q[..., 5] / rho - u2 * u2
    return rho, u1, u2, t11, t12, t22, 0.5 * (t11 + t22)


class Problem1D:
    def __init__(self, mesh, bc, eps, model):
        sx, = mesh.space
        vx, = mesh.velocity
        self.nx, self.nv = sx.n, vx.n
        self.dx = (sx.max - sx.min) / sx.n
        self.v = _c64(_centers(vx))
        faces = (bc.left, bc.right)
        self.face = [_face_code(f) for f in faces]
        self.wall_T = [getattr(f, "temperature", 0.0) for f in faces]
        self.tau_kind = TAU_KINDS[model.kind]
        self.tau_value = float(getattr(model, "value", 1.0))
        self.eps = float(eps)

    def cfg(self):
        c = _Cfg1D()
        c.nx, c.nv, c.dx = self.nx, self.nv, self.dx
        c.v = _p(self.v)
        for f in range(2):
            c.face[f] = self.face[f]
            c.wall_T[f] = self.wall_T[f]
        c.tau_kind, c.tau_value, c.eps = self.tau_kind, self.tau_value, self.eps
        return c


def step_1d_arrays(prob: Problem1D, Q, G, dt, src=None, qsrc=None):
    Q = _c64(Q)
    G = _c64(G)
    Qo = np.empty_like(Q)
    Go = np.empty_like(G)
    H = np.empty(prob.nx)
    err = _Err()
    s = _c64(src) if src is not None else None
    qs = _c64(qsrc) if qsrc is not None else None
    cfg = prob.cfg()
    rc = lib().mmo_step_1d(C.byref(cfg), _p(Q), _p(G), C.c_double(dt),
                           _p(s) if s is not None else None,
                           _p(qs) if qs is not None else None,
                           _p(Qo), _p(Go), _p(H), C.byref(err))
    if rc != 0:
        raise OracleStateError(ERR_MESSAGES.get(err.code, "invalid state"),
                               (err.i,), err.value)
    return Qo, Go, H


# ---------------------------------------------------------------------------
# The 10-function kernel contract (_kernels/_fallback.py), as NumPy
# restatements: the checker for the device plugin API.
# ---------------------------------------------------------------------------

def k_upwind_z_1d(G_ext, v, dx):
    """_fallback.py:27-32"""
    vm = np.minimum(v, 0.0)
    vp = np.maximum(v, 0.0)
    return (vm * (G_ext[2:] - G_ext[1:-1]) + vp * (G_ext[1:-1] - G_ext[:-2])) / dx


def k_project_field_1d(F, M, rho, u, T, v, dv):
    """_fallback.py:35-44"""
    w = (v[None, :] - u[:, None]) / np.sqrt(T)[:, None]
    b3 = np.sqrt(2.0) * (0.5 * w * w - 0.5)
    s = dv / rho
    a1 = s * F.sum(axis=1)
    a2 = s * (F * w).sum(axis=1)
    a3 = s * (F * b3).sum(axis=1)
    return (a1[:, None] + w * a2[:, None] + b3 * a3[:, None]) * M


def k_maxwellian_field_2d(rho, u1, u2, T, v1, v2):
    """_fallback.py:51-61"""
    w1 = v1[None, None, :, None] - u1[:, :, None, None]
    w2 = v2[None, None, None, :] - u2[:, :, None, None]
    Tf = T[:, :, None, None]
    return rho[:, :, None, None] / (2.0 * np.pi * Tf) * np.exp(-(w1 * w1 + w2 * w2) / (2.0 * Tf))


def k_project_field_2d(F, M, rho, u1, u2, T, v1, v2, dv):
    """_fallback.py:64-76"""
    st = np.sqrt(T)[:, :, None, None]
    w1 = (v1[None, None, :, None] - u1[:, :, None, None]) / st
    w2 = (v2[None, None, None, :] - u2[:, :, None, None]) / st
    b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0
    s = (dv / rho)[:, :, None, None]
    a1 = s * F.sum(axis=(2, 3), keepdims=True)
    a2 = s * (F * w1).sum(axis=(2, 3), keepdims=True)
    a3 = s * (F * w2).sum(axis=(2, 3), keepdims=True)
    a4 = s * (F * b4).sum(axis=(2, 3), keepdims=True)
    return (a1 + w1 * a2 + w2 * a3 + b4 * a4) * M


def k_transport_stage_2d(G_ext, M, rho, u1, u2, T, v1, v2, d, dt, axis):
    """_fallback.py:79-101"""
    if axis == 0:
        vm = np.minimum(v1, 0.0)[None, None, :, None]
        vp = np.maximum(v1, 0.0)[None, None, :, None]
        G = G_ext[1:-1]
        Z = (vm * (G_ext[2:] - G) + vp * (G - G_ext[:-2])) / d
    else:
        vm = np.minimum(v2, 0.0)[None, None, None, :]
        vp = np.maximum(v2, 0.0)[None, None, None, :]
        G = G_ext[:, 1:-1]
        Z = (vm * (G_ext[:, 2:] - G) + vp * (G - G_ext[:, :-2])) / d
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    Zhat = k_project_field_2d(Z, M, rho, u1, u2, T, v1, v2, dv)
    return G - dt * (Z - Zhat)


def k_ghat_2d(M, rho, u1, u2, T, s11, s12, gT1, gT2, tau, v1, v2):
    """_fallback.py:104-123"""
    w1 = v1[None, None, :, None] - u1[:, :, None, None]
    w2 = v2[None, None, None, :] - u2[:, :, None, None]
    Tf = T[:, :, None, None]
    e = (lambda a: a[:, :, None, None])
    bs = (-w2 * w2 * e(s11) + 2.0 * w1 * w2 * e(s12) + w1 * w1 * e(s11)) / (2.0 * Tf)
    cfac = (w1 * w1 + w2 * w2) / (2.0 * Tf) - 2.0
    cg = cfac * (w1 * e(gT1) + w2 * e(gT2)) / Tf
    return -(bs + cg) * M / e(tau)


def k_add_gaussian_term_2d(Ghat, M, rho, u1, u2, m11, m12, m22, eps, v1, v2):
    """_fallback.py:126-137 (returns a new array)"""
    e = (lambda a: a[:, :, None, None])
    c11, c12, c22 = e(m11), e(m12), e(m22)
    det = c11 * c22 - c12 * c12
    w1 = v1[None, None, :, None] - u1[:, :, None, None]
    w2 = v2[None, None, None, :] - u2[:, :, None, None]
    quad = (c22 * w1 * w1 - 2.0 * c12 * w1 * w2 + c11 * w2 * w2) / det
    Gs = e(rho) / (2.0 * np.pi * np.sqrt(det)) * np.exp(-0.5 * quad)
    return Ghat + (Gs - M) / eps


def k_add_lowrank_4d(out, coeffs, shapes):
    """_fallback.py:140-144 (returns a new array)"""
    out = np.array(out, copy=True)
    for c, s in zip(coeffs, shapes):
        out += c[:, :, None, None] * s[None, None, :, :]
    return out


def k_relax_2d(G, Ghat, tau, dt, eps):
    """_fallback.py:147-157"""
    denom = eps + dt * tau
    return (eps / denom)[:, :, None, None] * G + (dt * tau / denom)[:, :, None, None] * Ghat


def k_heat_tensor_2d(G, u1, u2, v1, v2, dv, eps):
    """_fallback.py:160-173"""
    w1 = v1[None, None, :, None] - u1[:, :, None, None]
    w2 = v2[None, None, None, :] - u2[:, :, None, None]
    f = eps * dv
    return (f * (w1 ** 3 * G).sum(axis=(2, 3)), f * (w1 * w1 * w2 * G).sum(axis=(2, 3)),
            f * (w1 * w2 * w2 * G).sum(axis=(2, 3)), f * (w2 ** 3 * G).sum(axis=(2, 3)))


if os.environ.get("MM_ORACLE_THREADS"):
    set_num_threads(int(os.environ["MM_ORACLE_THREADS"]))

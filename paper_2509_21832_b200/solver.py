"""Device-resident time stepper: the drop-in for the reference's hot path.

Reference interfaces mirrored here:
  State2D, step_2d, run_2d       pkg/src/micromacro/runner/loop.py:75-129
  heat_flux_tensor_2d            pkg/src/micromacro/macro2d.py:23-29
  frame moments (H with u^{n+1}) pkg/src/micromacro/runner/cases.py:167-176

``step_2d`` keeps the reference's functional contract -- it returns a new
State2D and never mutates its input -- but the returned state lives in HBM:
``state.Q`` / ``state.G`` download lazily (and raise a pending
InvalidStateError first), so a loop of ``step_2d`` calls never round-trips
the 4-D micro field through the host.  All arithmetic runs in libmm2d.so
(csrc/); PyTorch is used only for device memory and stream plumbing.
"""

from __future__ import annotations

import ctypes as C
from collections import OrderedDict

import numpy as np

from . import _native
from .boundary import face_code, is_wall
from .errors import ConfigurationError, InvalidStateError, NativeLibraryError
from .gas_state import TAU_KIND_CODES, conserved_2d
from .mesh import PhaseMesh, cell_centers, plan_time


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise NativeLibraryError("PyTorch is required for device buffers") from exc
    if not torch.cuda.is_available():
        raise NativeLibraryError("a CUDA device is required: the solver has no CPU path")
    return torch


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream_handle(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_config(mesh: PhaseMesh, bc, eps, model, grid=(1, 1), rank=(0, 0), device=0):
    """Fill the POD ``mm2d_config`` from the reference-style problem objects
    (duck-typed: the reference's own Axis/BoundarySpec2D/CollisionModel work)."""
    if len(mesh.space) != 2:
        raise ConfigurationError("the 2D solver needs a 2D2V PhaseMesh")
    sx, sy = mesh.space
    vx, vy = mesh.velocity
    cfg = _native.Config()
    cfg.nx, cfg.ny = int(sx.n), int(sy.n)
    cfg.x_min, cfg.x_max, cfg.y_min, cfg.y_max = sx.min, sx.max, sy.min, sy.max
    cfg.nv1, cfg.nv2 = int(vx.n), int(vy.n)
    cfg.v1_min, cfg.v1_max, cfg.v2_min, cfg.v2_max = vx.min, vx.max, vy.min, vy.max
    for f, face in enumerate((bc.left, bc.right, bc.bottom, bc.top)):
        cfg.face[f] = face_code(face)
        cfg.wall_T[f] = float(face.temperature) if is_wall(face) else 0.0
        cfg.wall_U[f] = float(getattr(face, "velocity", 0.0)) if is_wall(face) else 0.0
    if model.kind not in TAU_KIND_CODES:
        raise ConfigurationError(f"unknown collision model kind {model.kind!r}")
    cfg.tau_kind = TAU_KIND_CODES[model.kind]
    cfg.tau_value = float(getattr(model, "value", 1.0))
    cfg.nu = float(model.nu)
    cfg.eps = float(eps)
    cfg.px, cfg.py = int(grid[0]), int(grid[1])
    cfg.rx, cfg.ry = int(rank[0]), int(rank[1])
    cfg.device = int(device)
    return cfg


class Solver2D:
    """One libmm2d context: a (mesh, bc, eps, model) problem on one GPU,
    optionally one block of a px x py decomposition."""

    def __init__(self, mesh, bc, eps, model, grid=(1, 1), rank=(0, 0), device=None):
        torch = _torch()
        self.torch = torch
        self.lib = _native.load()
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", int(device))
        self.mesh, self.bc, self.eps, self.model = mesh, bc, float(eps), model
        self.grid, self.rank = tuple(grid), tuple(rank)
        self.cfg = make_config(mesh, bc, eps, model, grid, rank, self.device.index)
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            rc = self.lib.mm2d_create(C.byref(self.cfg), C.byref(ctx))
        if rc != _native.OK:
            raise ConfigurationError(f"mm2d_create failed (code {rc})")
        self.ctx = ctx
        bx, by, i0, j0 = (C.c_int() for _ in range(4))
        self.lib.mm2d_block(ctx, C.byref(bx), C.byref(by), C.byref(i0), C.byref(j0))
        self.bx, self.by, self.i0, self.j0 = bx.value, by.value, i0.value, j0.value
        self.nv1, self.nv2 = self.cfg.nv1, self.cfg.nv2
        self.V = self.nv1 * self.nv2
        self.v1 = cell_centers(mesh.velocity[0])
        self.v2 = cell_centers(mesh.velocity[1])

    # -- plumbing ---------------------------------------------------------
    def _rc(self, rc):
        if rc == _native.OK:
            return
        msg = _native.last_error(self.ctx)
        if rc == _native.ERR_CONFIG:
            raise ConfigurationError(msg)
        if rc == _native.ERR_STATE:
            self.check()
        raise RuntimeError(f"libmm2d failure (code {rc}): {msg}")

    def empty_state(self):
        t = self.torch
        Q = t.empty((self.bx, self.by, 6), dtype=t.float64, device=self.device)
        G = t.empty((self.bx, self.by, self.nv1, self.nv2), dtype=t.float64, device=self.device)
        return Q, G

    def to_device(self, a, shape):
        t = self.torch
        if isinstance(a, t.Tensor):
            a = a.to(device=self.device, dtype=t.float64)
        else:
            a = t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        if tuple(a.shape) != tuple(shape):
            raise ConfigurationError(f"array shape {tuple(a.shape)} != expected {tuple(shape)}")
        return a.contiguous()

    # -- the step ---------------------------------------------------------
    def step(self, Q, G, dt, Q_out=None, G_out=None, H_out=None, src=None, qsrc=None):
        """One step_2d on device tensors; returns (Q_new, G_new, H) where H is
        the (4, bx, by) heat tensor taken with u^n inside the step."""
        t = self.torch
        if Q_out is None or G_out is None:
            Q_out, G_out = self.empty_state()
        if H_out is None:
            H_out = t.empty((4, self.bx, self.by), dtype=t.float64, device=self.device)
        nsrc, sc, ss, qs = 0, None, None, None
        if src is not None:
            coeffs, shapes = src
            sc = self.to_device(coeffs, np.shape(coeffs))
            ss = self.to_device(shapes, np.shape(shapes))
            nsrc = int(sc.shape[0])
        if qsrc is not None:
            qs = self.to_device(qsrc, (self.bx, self.by, 6))
        with t.cuda.device(self.device):
            rc = self.lib.mm2d_step(self.ctx, _ptr(Q), _ptr(G), C.c_double(dt), _ptr(Q_out),
                                    _ptr(G_out), _ptr(H_out), nsrc, _ptr(sc), _ptr(ss),
                                    _ptr(qs), _stream_handle(t))
        self._rc(rc)
        # keep source buffers alive until the stream has consumed them
        self._pending_src = (sc, ss, qs)
        return Q_out, G_out, H_out

    def run(self, Q, G, dt, n_steps, H_out=None, Q_b=None, G_b=None):
        """n_steps steps replayed from a captured CUDA graph (ping-pong
        between (Q, G) and (Q_b, G_b)); returns the final (Q, G)."""
        t = self.torch
        if Q_b is None or G_b is None:
            Q_b, G_b = self.empty_state()
        with t.cuda.device(self.device):
            self._rc(self.lib.mm2d_attach_state(self.ctx, _ptr(Q), _ptr(G), _ptr(Q_b),
                                                _ptr(G_b), _ptr(H_out)))
            self._rc(self.lib.mm2d_set_stream(self.ctx, _stream_handle(t)))
            self._rc(self.lib.mm2d_run(self.ctx, C.c_double(dt), int(n_steps)))
        cur = self.lib.mm2d_current_index(self.ctx)
        return (Q, G) if cur == 0 else (Q_b, G_b)

    def heat_tensor(self, G, Q):
        """(4, bx, by) heat tensor of G about the velocity of Q."""
        t = self.torch
        H = t.empty((4, self.bx, self.by), dtype=t.float64, device=self.device)
        with t.cuda.device(self.device):
            self._rc(self.lib.mm2d_heat_tensor(self.ctx, _ptr(G), _ptr(Q), _ptr(H),
                                               _stream_handle(t)))
        return H

    def check(self):
        """Raise the pending InvalidStateError, if any (synchronises)."""
        kind, i, j, val = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        with self.torch.cuda.device(self.device):
            rc = self.lib.mm2d_check(self.ctx, C.byref(kind), C.byref(i), C.byref(j),
                                     C.byref(val))
        if rc == _native.OK:
            return
        if rc == _native.ERR_STATE:
            raise InvalidStateError(_native.STATE_MESSAGES.get(kind.value, "invalid state"),
                                    cell=(i.value, j.value), value=val.value)
        raise RuntimeError(f"libmm2d failure (code {rc}): {_native.last_error(self.ctx)}")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mm2d_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_CACHE: "OrderedDict[tuple, Solver2D]" = OrderedDict()
_CACHE_SIZE = 4


def get_solver(mesh, bc, eps, model, device=None) -> Solver2D:
    """Solver for a problem, cached by its (hashable, frozen) description."""
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else int(device)
    try:
        key = (mesh, bc, float(eps), model, dev)
        hash(key)
    except TypeError:
        key = None
    if key is not None and key in _CACHE:
        _CACHE.move_to_end(key)
        return _CACHE[key]
    s = Solver2D(mesh, bc, eps, model, device=dev)
    if key is not None:
        _CACHE[key] = s
        while len(_CACHE) > _CACHE_SIZE:
            # drop only the cache's reference: states returned by step_2d /
            # run_2d keep their solver (and its pending error) alive, and
            # __del__ frees the context once nothing refers to it
            _CACHE.popitem(last=False)
    return s


class State2D:
    """Drop-in for the reference's ``State2D(t, Q, G)`` dataclass
    (loop.py:75-79).  Q (nx, ny, 6) and G (nx, ny, nv1, nv2) may be host
    NumPy arrays or device tensors; reading ``.Q`` / ``.G`` returns NumPy
    (downloaded once, after raising any pending device error)."""

    __slots__ = ("t", "_Q", "_G", "_Qh", "_Gh", "_solver", "H_step")

    def __init__(self, t, Q, G, _solver=None, H_step=None):
        self.t = t
        self._solver = _solver
        self._Q = Q
        self._G = G
        self._Qh = None
        self._Gh = None
        self.H_step = H_step

    @staticmethod
    def _is_dev(a):
        return hasattr(a, "is_cuda") and a.is_cuda

    def _host(self, a, cache_name):
        if not self._is_dev(a):
            return a
        cached = getattr(self, cache_name)
        if cached is None:
            if self._solver is not None:
                self._solver.check()
            cached = a.detach().cpu().numpy()
            setattr(self, cache_name, cached)
        return cached

    @property
    def Q(self):
        return self._host(self._Q, "_Qh")

    @Q.setter
    def Q(self, value):
        self._Q, self._Qh = value, None

    @property
    def G(self):
        return self._host(self._G, "_Gh")

    @G.setter
    def G(self, value):
        self._G, self._Gh = value, None

    def device_arrays(self, solver: Solver2D):
        """(Q, G) as device tensors on the solver's GPU (uploading host data)."""
        if self._solver is not None and self._solver is not solver and self._is_dev(self._Q):
            self._solver.check()
        Q = solver.to_device(self._Q, (solver.bx, solver.by, 6))
        G = solver.to_device(self._G, (solver.bx, solver.by, solver.nv1, solver.nv2))
        return Q, G

    def __repr__(self):
        where = "device" if self._is_dev(self._G) else "host"
        return f"State2D(t={self.t!r}, Q={tuple(self._Q.shape)}, G={tuple(self._G.shape)}, {where})"


def step_2d(state, mesh, bc, eps, model, dt, micro_source=None, macro_source=None) -> State2D:
    """One step: split micro update, heat tensor with u^n, Strang-split
    macro update (loop.py:82-111), fused on the GPU.

    micro_source(t, x, y, v1, v2) -> (coeffs, shapes) low-rank projected
    source; macro_source(t, x, y) -> (nx, ny, 6) moment source; both at t^n.
    """
    solver = get_solver(mesh, bc, eps, model)
    if isinstance(state, State2D):
        st = state
    else:  # the reference's own State2D (or any object with t, Q, G)
        st = State2D(state.t, state.Q, state.G)
    # no host synchronisation here: a state stepped on the same context keeps
    # any pending device error sticky (the step's kernels skip their work and
    # the error is raised when the host next reads .Q / .G or calls check());
    # a state from another context is checked in device_arrays
    Q, G = st.device_arrays(solver)
    src = qsrc = None
    if micro_source is not None or macro_source is not None:
        x = cell_centers(mesh.space[0])
        y = cell_centers(mesh.space[1])
        if micro_source is not None:
            src = micro_source(st.t, x, y, solver.v1, solver.v2)
        if macro_source is not None:
            qsrc = macro_source(st.t, x, y)
    Qn, Gn, H = solver.step(Q, G, dt, src=src, qsrc=qsrc)
    return State2D(st.t + dt, Qn, Gn, _solver=solver, H_step=H)


def run_2d(mesh, bc, eps, model, rho0, u10, u20, t11_0, t12_0, t22_0, G0, t_final, cfl,
           micro_source=None, macro_source=None, on_step=None):
    """Run from primitive initial data to t_final with plan_time's constant
    step (loop.py:114-129); returns (State2D, TimePlan).  Without sources or
    callbacks the whole loop is one CUDA-graph replay on the device."""
    plan = plan_time(t_final, cfl, mesh)
    Q0 = conserved_2d(rho0, u10, u20, t11_0, t12_0, t22_0)
    state = State2D(0.0, Q0, np.array(G0, dtype=float))
    if micro_source is None and macro_source is None and on_step is None:
        solver = get_solver(mesh, bc, eps, model)
        Q, G = state.device_arrays(solver)
        Qf, Gf = solver.run(Q, G, plan.dt, plan.n_steps)
        return State2D(plan.n_steps * plan.dt, Qf, Gf, _solver=solver), plan
    for n in range(plan.n_steps):
        state = step_2d(state, mesh, bc, eps, model, plan.dt, micro_source=micro_source,
                        macro_source=macro_source)
        state.t = (n + 1) * plan.dt
        if on_step is not None:
            on_step(n, state)
    return state, plan


def frame_moments(state: State2D, mesh, bc, eps, model):
    """The frame_2d moment set (cases.py:167-176; frames.py:31-33):
    rho mom1 mom2 e11 e12 e22 h111 h112 h122 h222, with H taken about the
    velocity of the frame's own Q (u^{n+1}), as (10, nx, ny) NumPy."""
    solver = get_solver(mesh, bc, eps, model)
    Q, G = state.device_arrays(solver)
    H = solver.heat_tensor(G, Q)
    Qh = Q.cpu().numpy()
    return np.concatenate([np.moveaxis(Qh, -1, 0), H.cpu().numpy()], axis=0)


__all__ = ["Solver2D", "State2D", "get_solver", "step_2d", "run_2d", "frame_moments",
           "make_config"]

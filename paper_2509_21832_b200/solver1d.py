"""Device-resident 1D1V stepper (BASELINE config 1).

Reference interfaces mirrored here:
  State1D, step_1d, run_1d      pkg/src/micromacro/runner/loop.py:24-72
  heat_flux_1d (the H output)   pkg/src/micromacro/macro1d.py:16-19

Same contract as the 2D solver (solver.py): ``step_1d`` returns a new
State1D without mutating its input, the arrays live in HBM and download
lazily, and a pending InvalidStateError (primitives_1d, gas_state.py:44-54)
is raised on that download.  ``run_1d`` without sources or callbacks is ONE
launch of the cluster-resident kernel (csrc/mm1d_resident.cuh) when the
state fits in a cluster's shared memory, else a CUDA-graph replay of the
two-kernel step.  All arithmetic runs in libmm2d.so (C ABI: include/mm1d.h).
"""

from __future__ import annotations

import ctypes as C
from collections import OrderedDict

import numpy as np

from . import _native
from .boundary import face_code, is_wall
from .errors import ConfigurationError, InvalidStateError
from .gas_state import TAU_KIND_CODES, conserved_1d
from .mesh import cell_centers, plan_time
from .solver import _ptr, _stream_handle, _torch


def make_config_1d(mesh, bc, eps, model, device=0):
    """Fill the POD ``mm1d_config`` from reference-style problem objects."""
    if len(mesh.space) != 1 or len(mesh.velocity) != 1:
        raise ConfigurationError("the 1D solver needs a 1D1V PhaseMesh")
    sx, = mesh.space
    vx, = mesh.velocity
    cfg = _native.Config1D()
    cfg.nx, cfg.x_min, cfg.x_max = int(sx.n), float(sx.min), float(sx.max)
    cfg.nv, cfg.v_min, cfg.v_max = int(vx.n), float(vx.min), float(vx.max)
    for f, face in enumerate((bc.left, bc.right)):
        cfg.face[f] = face_code(face)
        cfg.wall_T[f] = float(face.temperature) if is_wall(face) else 0.0
    if model.kind not in TAU_KIND_CODES:
        raise ConfigurationError(f"unknown collision model kind {model.kind!r}")
    cfg.tau_kind = TAU_KIND_CODES[model.kind]
    cfg.tau_value = float(getattr(model, "value", 1.0))
    cfg.eps = float(eps)
    cfg.device = int(device)
    return cfg


class Solver1D:
    """One mm1d context: a (mesh, bc, eps, model) 1D problem on one GPU."""

    def __init__(self, mesh, bc, eps, model, device=None):
        torch = _torch()
        self.torch = torch
        self.lib = _native.load()
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", int(device))
        self.mesh, self.bc, self.eps, self.model = mesh, bc, float(eps), model
        self.cfg = make_config_1d(mesh, bc, eps, model, self.device.index)
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            rc = self.lib.mm1d_create(C.byref(self.cfg), C.byref(ctx))
        if rc != _native.OK:
            msg = self.lib.mm1d_last_error(ctx) if ctx else b""
            raise ConfigurationError(f"mm1d_create failed (code {rc}) {msg!r}")
        self.ctx = ctx
        self.nx, self.nv = self.cfg.nx, self.cfg.nv
        self.v = cell_centers(mesh.velocity[0])
        self.resident = bool(self.lib.mm1d_resident(ctx))

    def _rc(self, rc):
        if rc == _native.OK:
            return
        m = self.lib.mm1d_last_error(self.ctx)
        msg = m.decode() if m else ""
        if rc == _native.ERR_CONFIG:
            raise ConfigurationError(msg)
        if rc == _native.ERR_STATE:
            self.check()
        raise RuntimeError(f"libmm2d (1D) failure (code {rc}): {msg}")

    def to_device(self, a, shape):
        t = self.torch
        if isinstance(a, t.Tensor):
            a = a.to(device=self.device, dtype=t.float64)
        else:
            a = t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        if tuple(a.shape) != tuple(shape):
            raise ConfigurationError(f"array shape {tuple(a.shape)} != expected {tuple(shape)}")
        return a.contiguous()

    def empty_state(self):
        t = self.torch
        return (t.empty((self.nx, 3), dtype=t.float64, device=self.device),
                t.empty((self.nx, self.nv), dtype=t.float64, device=self.device))

    def step(self, Q, G, dt, Q_out=None, G_out=None, H_out=None, src=None, qsrc=None):
        """One step_1d on device tensors; returns (Q_new, G_new, H) with H the
        heat_flux_1d of G_new."""
        t = self.torch
        if Q_out is None or G_out is None:
            Q_out, G_out = self.empty_state()
        if H_out is None:
            H_out = t.empty((self.nx,), dtype=t.float64, device=self.device)
        s = self.to_device(src, (self.nx, self.nv)) if src is not None else None
        qs = self.to_device(qsrc, (self.nx, 3)) if qsrc is not None else None
        with t.cuda.device(self.device):
            rc = self.lib.mm1d_step(self.ctx, _ptr(Q), _ptr(G), C.c_double(dt), _ptr(Q_out),
                                    _ptr(G_out), _ptr(H_out), _ptr(s), _ptr(qs),
                                    _stream_handle(t))
        self._rc(rc)
        self._pending_src = (s, qs)
        return Q_out, G_out, H_out

    def run_host(self, Q, G, dt, n_steps):
        """run_1d's loop on context-owned state: host (Q, G) in, n_steps on
        the device, host (Q, G, H) out.  Raises a pending InvalidStateError."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        G = np.ascontiguousarray(G, dtype=np.float64)
        if Q.shape != (self.nx, 3) or G.shape != (self.nx, self.nv):
            raise ConfigurationError("state shapes do not match the mesh")
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        with self.torch.cuda.device(self.device):
            self._rc(self.lib.mm1d_upload(self.ctx, p(Q), p(G)))
            self._rc(self.lib.mm1d_run(self.ctx, C.c_double(dt), int(n_steps)))
            Qo, Go, Ho = np.empty_like(Q), np.empty_like(G), np.empty(self.nx)
            self._rc(self.lib.mm1d_download(self.ctx, p(Qo), p(Go), p(Ho)))
        self.check()
        return Qo, Go, Ho

    def check(self):
        """Raise the pending InvalidStateError, if any (synchronises)."""
        kind, i, val = C.c_int(), C.c_int(), C.c_double()
        with self.torch.cuda.device(self.device):
            rc = self.lib.mm1d_check(self.ctx, C.byref(kind), C.byref(i), C.byref(val))
        if rc == _native.OK:
            return
        if rc == _native.ERR_STATE:
            raise InvalidStateError(_native.STATE_MESSAGES.get(kind.value, "invalid state"),
                                    cell=(i.value,), value=val.value)
        raise RuntimeError(f"libmm2d (1D) failure (code {rc})")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mm1d_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_CACHE: "OrderedDict[tuple, Solver1D]" = OrderedDict()


def get_solver_1d(mesh, bc, eps, model, device=None) -> Solver1D:
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
    s = Solver1D(mesh, bc, eps, model, device=dev)
    if key is not None:
        _CACHE[key] = s
        while len(_CACHE) > 4:
            # drop only the cache's reference: live states keep their solver
            _CACHE.popitem(last=False)
    return s


class State1D:
    """Drop-in for the reference's ``State1D(t, Q, G)`` (loop.py:24-28);
    Q (nx, 3) and G (nx, nv) may be host arrays or device tensors."""

    __slots__ = ("t", "_Q", "_G", "_Qh", "_Gh", "_solver", "H_step")

    def __init__(self, t, Q, G, _solver=None, H_step=None):
        self.t = t
        self._solver = _solver
        self._Q, self._G = Q, G
        self._Qh = self._Gh = None
        self.H_step = H_step

    def _host(self, a, cache_name):
        if not (hasattr(a, "is_cuda") and a.is_cuda):
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

    def device_arrays(self, solver: Solver1D):
        if self._solver is not None and self._solver is not solver:
            self._solver.check()
        return (solver.to_device(self._Q, (solver.nx, 3)),
                solver.to_device(self._G, (solver.nx, solver.nv)))

    def __repr__(self):
        return f"State1D(t={self.t!r}, Q={tuple(self._Q.shape)}, G={tuple(self._G.shape)})"


def step_1d(state, mesh, bc, eps, model, dt, micro_source=None, macro_source=None) -> State1D:
    """One step: micro update, heat-flux moment, macro update (loop.py:31-51).

    micro_source(t, x, v) -> (nx, nv) projected residual; macro_source(t, x)
    -> (nx, 3) moment source; both evaluated at t^n.
    """
    solver = get_solver_1d(mesh, bc, eps, model)
    st = state if isinstance(state, State1D) else State1D(state.t, state.Q, state.G)
    # no per-step host sync: errors stay sticky on the context and surface
    # when the host reads the state (device_arrays checks a foreign context)
    Q, G = st.device_arrays(solver)
    x = cell_centers(mesh.space[0])
    src = micro_source(st.t, x, solver.v) if micro_source is not None else None
    qsrc = macro_source(st.t, x) if macro_source is not None else None
    Qn, Gn, H = solver.step(Q, G, dt, src=src, qsrc=qsrc)
    return State1D(st.t + dt, Qn, Gn, _solver=solver, H_step=H)


def run_1d(mesh, bc, eps, model, rho0, u0, T0, G0, t_final, cfl, micro_source=None,
           macro_source=None, on_step=None):
    """Run from primitive initial data to t_final with plan_time's constant
    step (loop.py:54-72); returns (State1D, TimePlan)."""
    plan = plan_time(t_final, cfl, mesh)
    Q0 = conserved_1d(rho0, u0, T0)
    if micro_source is None and macro_source is None and on_step is None:
        solver = get_solver_1d(mesh, bc, eps, model)
        Q, G, H = solver.run_host(Q0, np.array(G0, dtype=float), plan.dt, plan.n_steps)
        return State1D(plan.n_steps * plan.dt, Q, G, H_step=H), plan
    state = State1D(0.0, Q0, np.array(G0, dtype=float))
    for n in range(plan.n_steps):
        state = step_1d(state, mesh, bc, eps, model, plan.dt, micro_source=micro_source,
                        macro_source=macro_source)
        state.t = (n + 1) * plan.dt
        if on_step is not None:
            on_step(n, state)
    return state, plan


__all__ = ["Solver1D", "State1D", "get_solver_1d", "step_1d", "run_1d", "make_config_1d"]

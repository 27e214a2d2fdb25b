"""Run driver with frame capture and steady-state tracking, device-resident
(drop-in for the reference's ``_advance`` / ``run_single_2d`` time loop,
pkg/src/micromacro/runner/cases.py:188-256, and ``totals`` 178-182).

The loop semantics are the reference's: a fixed step from ``plan_time``, an
optional step cap, frames captured at the steps nearest the requested
times, and the maximum |Q^{n+1} - Q^n| over the last 10% of steps.  The
state never leaves HBM: step ranges between events are CUDA-graph replays
(``Solver2D.run``), the steady-state maximum is accumulated on the device by
``mm2d_max_abs_diff`` (read once at the end), and a frame costs one heat
tensor launch plus the download the snapshot itself asks for.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from ..mesh import plan_time


@dataclass
class RunRecord:
    """Same fields as the reference's ``RunRecord`` (cases.py:188-196)."""

    state: object
    plan: object
    seconds: float
    steps_run: int
    frames: list = field(default_factory=list)   # (time, snapshot(state))
    steady_max_change: float = float("nan")


def totals(Q, cell_volume):
    """Spatially integrated conserved moments (cases.py:178-182)."""
    Q = np.asarray(Q)
    return tuple(float(v) for v in Q.reshape(-1, Q.shape[-1]).sum(axis=0) * cell_volume)


def snap_steps(frame_times, dt, n_steps):
    """{step index (1-based): requested time}, the nearest step to each
    frame time clipped to [1, n_steps], first request winning
    (cases.py:209-212)."""
    out = {}
    for ft in frame_times:
        out.setdefault(int(np.clip(round(ft / dt), 1, n_steps)), ft)
    return out


def steady_window(n_steps):
    """Number of trailing steps tracked for the steady-state change."""
    return max(1, int(math.ceil(0.1 * n_steps)))


def advance_2d(mesh, bc, eps, model, state, t_final, cfl, frame_times=(), max_steps=None,
               micro_source=None, macro_source=None, snapshot=None, track_steady=False):
    """The reference's ``_advance`` for ``step_2d`` (cases.py:199-231).

    ``snapshot(state)`` is called with the live device state at each frame
    step and its result stored; ``frame_moments`` gives the reference's
    ``frame_2d`` moment set.  Returns a :class:`RunRecord`.
    """
    from ..solver import State2D, get_solver, step_2d

    plan = plan_time(t_final, cfl, mesh)
    n_steps = plan.n_steps
    if max_steps:
        n_steps = min(n_steps, int(max_steps))
    snaps = snap_steps(frame_times, plan.dt, n_steps)
    window = steady_window(n_steps)
    first_tracked = n_steps - window      # 0-based step index n >= this is tracked
    solver = get_solver(mesh, bc, eps, model)
    torch = solver.torch
    lib = solver.lib
    stream = C.c_void_p(torch.cuda.current_stream(solver.device).cuda_stream)
    dmax = torch.zeros(1, dtype=torch.float64, device=solver.device)
    captured = []

    def track(prev_Q, new_Q):
        rc = lib.mm2d_max_abs_diff(solver.ctx, C.c_void_p(prev_Q.data_ptr()),
                                   C.c_void_p(new_Q.data_ptr()), int(new_Q.numel()),
                                   C.c_void_p(dmax.data_ptr()), stream)
        solver._rc(rc)

    st = state if isinstance(state, State2D) else State2D(state.t, state.Q, state.G)
    t0 = time.perf_counter()
    if micro_source is not None or macro_source is not None:
        # sources are evaluated on the host at t^n: one step_2d per step
        for n in range(n_steps):
            prev = st
            st = step_2d(st, mesh, bc, eps, model, plan.dt, micro_source=micro_source,
                         macro_source=macro_source)
            st.t = (n + 1) * plan.dt
            if track_steady and n >= first_tracked:
                track(prev.device_arrays(solver)[0], st._Q)
            if snapshot is not None and (n + 1) in snaps:
                captured.append((snaps[n + 1], snapshot(st)))
    else:
        Qa, Ga = st.device_arrays(solver)
        Qa, Ga = Qa.clone(), Ga.clone()
        bufs = [(Qa, Ga), (torch.empty_like(Qa), torch.empty_like(Ga))]
        p = lambda t: C.c_void_p(t.data_ptr())
        with torch.cuda.device(solver.device):
            # one attachment for the whole run: the graphs stay captured and
            # mm2d_current_index says which buffer pair holds the state
            solver._rc(lib.mm2d_attach_state(solver.ctx, p(bufs[0][0]), p(bufs[0][1]),
                                             p(bufs[1][0]), p(bufs[1][1]), None))
            solver._rc(lib.mm2d_set_stream(solver.ctx, stream))
            # event steps: frames, and every step of the tracked window (the
            # step before the window ends a chunk so the window runs 1 by 1)
            events = set(snaps)
            if track_steady:
                events |= set(range(max(first_tracked, 1), n_steps + 1))
            done = 0
            for ev in sorted(events) + [n_steps]:
                k = ev - done
                if k <= 0:
                    continue
                prev = lib.mm2d_current_index(solver.ctx)
                solver._rc(lib.mm2d_run(solver.ctx, C.c_double(plan.dt), int(k)))
                cur = lib.mm2d_current_index(solver.ctx)
                done = ev
                if track_steady and done > first_tracked:
                    track(bufs[prev][0], bufs[cur][0])      # k == 1 inside the window
                if snapshot is not None and done in snaps:
                    live = State2D(done * plan.dt, bufs[cur][0], bufs[cur][1], _solver=solver)
                    captured.append((snaps[done], snapshot(live)))
        cur = lib.mm2d_current_index(solver.ctx)
        st = State2D(n_steps * plan.dt, bufs[cur][0], bufs[cur][1], _solver=solver)
    torch.cuda.synchronize(solver.device)
    seconds = time.perf_counter() - t0
    solver.check()
    steady = float(dmax.item()) if track_steady else float("nan")
    return RunRecord(state=st, plan=plan, seconds=seconds, steps_run=n_steps, frames=captured,
                     steady_max_change=steady)


__all__ = ["RunRecord", "advance_2d", "totals", "snap_steps", "steady_window"]

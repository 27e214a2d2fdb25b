"""The run-driver names of the reference's case module that sit on the hot
path (pkg/src/micromacro/runner/cases.py): ``RunRecord``, ``totals``,
``_advance`` and the ``frame_2d`` moment set.  Case registry, config files
and frame-file I/O stay out of scope."""

from __future__ import annotations

import numpy as np

from .drive import RunRecord, advance_2d, totals

FIELDS_2D = ("rho", "mom1", "mom2", "e11", "e12", "e22", "h111", "h112", "h122", "h222")


def frame_2d(state, mesh, eps, bc=None, model=None):
    """``frame_2d`` (cases.py:167-176): Q and the heat tensor about u^{n+1},
    as {field: (nx, ny) array} with the reference's field names
    (frames.py:31-33)."""
    from ..gas_state import CollisionModel
    from ..solver import frame_moments
    if bc is None:
        bc = getattr(state._solver, "bc", None) if getattr(state, "_solver", None) else None
    if bc is None:
        raise ValueError("frame_2d needs the boundary spec of the run (bc=...)")
    model = model if model is not None else CollisionModel("esbgk_2d")
    m = frame_moments(state, mesh, bc, eps, model)
    return {name: np.asarray(m[k]) for k, name in enumerate(FIELDS_2D)}


def _advance(cfg, mesh, bc, eps, model, state, stepper=None, micro_source=None,
             macro_source=None, snapshot=None, track_steady=False):
    """``_advance`` (cases.py:199-231) for 2D states: ``cfg`` supplies
    ``t_final``, ``cfl``, ``max_steps`` and ``frame_times``.  The step is
    always this package's device step (``stepper`` is accepted for
    signature compatibility)."""
    return advance_2d(mesh, bc, eps, model, state, cfg.t_final, cfg.cfl,
                      frame_times=getattr(cfg, "frame_times", ()) or (),
                      max_steps=getattr(cfg, "max_steps", None),
                      micro_source=micro_source, macro_source=macro_source,
                      snapshot=snapshot, track_steady=track_steady)


__all__ = ["RunRecord", "totals", "frame_2d", "_advance", "FIELDS_2D"]

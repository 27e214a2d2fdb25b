"""Time loops (drop-in for pkg/src/micromacro/runner/loop.py:24-129)."""

from ..solver import State2D, run_2d, step_2d
from ..solver1d import State1D, run_1d, step_1d

__all__ = ["State1D", "step_1d", "run_1d", "State2D", "step_2d", "run_2d"]

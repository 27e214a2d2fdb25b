"""Time loops (drop-in for pkg/src/micromacro/runner/loop.py:75-129)."""

from ..solver import State2D, run_2d, step_2d

__all__ = ["State2D", "step_2d", "run_2d"]

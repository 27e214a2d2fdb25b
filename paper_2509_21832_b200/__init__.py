"""B200-native micro-macro ES-BGK 2D2V timestep (arXiv 2509.21832).

Drop-in for the reference solver's hot path (``micromacro.runner.loop.step_2d``
and friends): the same problem objects and functional API, with the step
fused into hand-written sm_100a CUDA kernels (csrc/, C ABI in include/mm2d.h).
"""

from .boundary import (EXTRAPOLATE, EXTRAPOLATE_1D, PERIODIC, PERIODIC_1D, SPECULAR,
                       BoundarySpec1D, BoundarySpec2D, WallSpec)
from .errors import ConfigurationError, InvalidStateError, NativeLibraryError
from .gas_state import (CollisionModel, TempTensor2D, conserved_1d, conserved_2d,
                        primitives_1d, primitives_2d)
from .mesh import Axis, PhaseMesh, TimePlan, cell_centers, plan_time

__version__ = "0.1.0"


def __getattr__(name):
    # device-path names load lazily so that host-only use (and the CPU test
    # suite) does not need a GPU
    if name in ("State2D", "step_2d", "run_2d", "Solver2D", "frame_moments", "get_solver"):
        from . import solver
        return getattr(solver, name)
    if name in ("State1D", "step_1d", "run_1d", "Solver1D", "get_solver_1d"):
        from . import solver1d
        return getattr(solver1d, name)
    if name == "heat_flux_tensor_2d":
        from .macro2d import heat_flux_tensor_2d
        return heat_flux_tensor_2d
    if name == "run_parallel_2d":
        from .parallel import run_parallel_2d
        return run_parallel_2d
    raise AttributeError(name)


__all__ = ["Axis", "PhaseMesh", "TimePlan", "cell_centers", "plan_time", "PERIODIC",
           "EXTRAPOLATE", "SPECULAR", "PERIODIC_1D", "EXTRAPOLATE_1D", "WallSpec", "BoundarySpec1D",
           "BoundarySpec2D", "CollisionModel", "TempTensor2D", "conserved_1d",
           "conserved_2d", "primitives_1d", "primitives_2d", "ConfigurationError",
           "InvalidStateError", "NativeLibraryError", "State2D", "step_2d", "run_2d",
           "Solver2D", "frame_moments", "heat_flux_tensor_2d", "run_parallel_2d",
           "State1D", "step_1d", "run_1d", "Solver1D"]

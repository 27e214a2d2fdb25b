"""Boundary specifications (drop-in for pkg/src/micromacro/boundary.py:21-81).

Face kinds: ``PERIODIC`` (paired), ``EXTRAPOLATE`` (zero-gradient copy),
``WallSpec`` (diffusely reflecting wall at fixed temperature, optional
tangential velocity) and ``SPECULAR`` (specularly reflecting wall, 2D only).

``SPECULAR`` is an extension beyond the reference, which has diffuse walls
only (BASELINE config 4 asks for reflecting walls).  Every ghost is the
mirror image of the edge cell in the wall-normal velocity: micro ghosts take
the edge distribution at v_n -> -v_n, macro ghosts negate the normal
momentum and E12, heat ghosts negate the components odd in v_n.  It needs a
velocity axis symmetric about zero along the wall normal.  The ghost-cell rules themselves run on the device
(csrc/mm2d_prep.cuh, mm2d_micro.cuh, mm2d_macro.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigurationError

PERIODIC = "periodic"
EXTRAPOLATE = "extrapolate"
SPECULAR = "specular"


@dataclass(frozen=True)
class WallSpec:
    """Diffuse wall at ``temperature``, sliding tangentially at ``velocity``."""

    temperature: float
    velocity: float = 0.0

    def __post_init__(self):
        if self.temperature <= 0:
            raise ConfigurationError(
                f"wall temperature must be positive, got {self.temperature}")


def is_wall(face) -> bool:
    """Duck-typed wall test (accepts the reference's own WallSpec too)."""
    return isinstance(face, WallSpec) or (
        not isinstance(face, str) and hasattr(face, "temperature"))


def _validate_face(face):
    if face in (PERIODIC, EXTRAPOLATE, SPECULAR) or is_wall(face):
        return
    raise ConfigurationError(f"unknown boundary face {face!r}")


def _paired(a, b, what):
    if (a == PERIODIC) != (b == PERIODIC):
        raise ConfigurationError(f"periodic {what} must come in pairs")


@dataclass(frozen=True)
class BoundarySpec1D:
    left: object
    right: object

    def __post_init__(self):
        for f in (self.left, self.right):
            _validate_face(f)
            if f == SPECULAR:
                raise ConfigurationError("specular walls are supported in 2D only")
        _paired(self.left, self.right, "boundaries")


@dataclass(frozen=True)
class BoundarySpec2D:
    """Faces left/right (x) and bottom/top (y)."""

    left: object
    right: object
    bottom: object
    top: object

    def __post_init__(self):
        for f in (self.left, self.right, self.bottom, self.top):
            _validate_face(f)
        _paired(self.left, self.right, "x-boundaries")
        _paired(self.bottom, self.top, "y-boundaries")

    def transposed(self) -> "BoundarySpec2D":
        return BoundarySpec2D(left=self.bottom, right=self.top,
                              bottom=self.left, top=self.right)

    @property
    def faces(self):
        return (self.left, self.right, self.bottom, self.top)


PERIODIC_1D = BoundarySpec1D(PERIODIC, PERIODIC)
EXTRAPOLATE_1D = BoundarySpec1D(EXTRAPOLATE, EXTRAPOLATE)


def face_code(face) -> int:
    """0 periodic, 1 extrapolate, 2 wall, 3 specular (include/mm2d.h MM2D_FACE_*)."""
    if face == PERIODIC:
        return 0
    if face == EXTRAPOLATE:
        return 1
    if is_wall(face):
        return 2
    if face == SPECULAR:
        return 3
    raise ConfigurationError(f"unknown boundary face {face!r}")


__all__ = ["PERIODIC", "EXTRAPOLATE", "SPECULAR", "WallSpec", "BoundarySpec1D", "BoundarySpec2D",
           "PERIODIC_1D", "EXTRAPOLATE_1D", "face_code", "is_wall"]

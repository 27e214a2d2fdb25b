"""Error types of the drop-in API (reference: pkg/src/micromacro/errors.py:4-24).

``ConfigurationError`` is a ``ValueError`` for bad setups;
``InvalidStateError`` is a ``RuntimeError`` for non-physical macro states and
carries the offending cell and value.  On the device path the state checks
run inside the kernels and set a sticky error word that the host reads at the
next synchronisation point, so the exception surfaces there instead of at the
exact step (documented in DESIGN.md).
"""


class ConfigurationError(ValueError):
    """Invalid run configuration or model parameter."""


class InvalidStateError(RuntimeError):
    """Non-physical macro state (rho <= 0 or a non-SPD tensor)."""

    def __init__(self, message, cell=None, value=None):
        text = message
        if cell is not None:
            text += f" at cell {cell}"
        if value is not None:
            text += f" (value {value})"
        super().__init__(text)
        self.cell = cell
        self.value = value


class NativeLibraryError(ImportError):
    """libmm2d.so is missing or could not be loaded (no CPU fallback)."""

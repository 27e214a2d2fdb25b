"""Heat-flux moments of the micro field (drop-in for
pkg/src/micromacro/macro2d.py:23-34).  The macro update itself runs fused on
the device inside ``step_2d`` (csrc/mm2d_macro.cuh)."""

from __future__ import annotations

import numpy as np

from . import _kernels as K


def heat_flux_tensor_2d(G, u1, u2, v1, v2, eps):
    """(H111, H112, H122, H222) = eps dv1 dv2 sum (v-u)^3-moments of G."""
    dv = (v1[1] - v1[0]) * (v2[1] - v2[0])
    return K.heat_tensor_2d(G, u1, u2, v1, v2, dv, eps)


def heat_flux_vector_2d(h111, h112, h122, h222):
    """h = (H111 + H122, H112 + H222) / 2."""
    return 0.5 * (np.asarray(h111) + np.asarray(h122)), 0.5 * (np.asarray(h112) + np.asarray(h222))


__all__ = ["heat_flux_tensor_2d", "heat_flux_vector_2d"]

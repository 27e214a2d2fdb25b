"""The reference's kernel plugin API on the GPU.

Drop-in for ``micromacro._kernels`` (pkg/src/micromacro/_kernels/__init__.py:
20-61): the same ten functions with the same signatures and array layouts
(_fallback.py:8-11), computed by the sm_100a kernels in libmm2d.so
(csrc/mm2d_contract.cuh).  Host NumPy arrays are copied to the device and the
results copied back; device tensors are used in place.  There is exactly one
backend -- no environment switch and no CPU fallback.

The fused timestep (solver.step_2d) does not go through these functions;
they serve callers of the kernel-level API and the unit-parity tests
(mirroring the reference's pkg/tests/test_kernels.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .solver import _torch

backend_name = "cuda-sm_100a"


def _lib():
    return _native.load()


def _dev(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _p(t):
    return C.c_void_p(t.data_ptr())


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _out(shape):
    torch = _torch()
    return torch.empty(shape, dtype=torch.float64, device="cuda")


def _host(t):
    return t.cpu().numpy()


def _check(rc):
    if rc != _native.OK:
        raise RuntimeError(f"libmm2d kernel failed (code {rc})")


def upwind_z_1d(G_ext, v, dx):
    G = _dev(G_ext)
    vv = _dev(v)
    nx, nv = G.shape[0] - 2, G.shape[1]
    Z = _out((nx, nv))
    _check(_lib().mm2d_k_upwind_z_1d(nx, nv, _p(G), _p(vv), C.c_double(dx), _p(Z), _stream()))
    return _host(Z)


def project_field_1d(F, M, rho, u, T, v, dv):
    F, M, rho, u, T, v = (_dev(a) for a in (F, M, rho, u, T, v))
    nx, nv = F.shape
    out = _out((nx, nv))
    _check(_lib().mm2d_k_project_field_1d(nx, nv, _p(F), _p(M), _p(rho), _p(u), _p(T), _p(v),
                                          C.c_double(dv), _p(out), _stream()))
    return _host(out)


def maxwellian_field_2d(rho, u1, u2, T, v1, v2, out=None):
    rho, u1, u2, T, v1, v2 = (_dev(a) for a in (rho, u1, u2, T, v1, v2))
    nx, ny = rho.shape
    M = _out((nx, ny, v1.shape[0], v2.shape[0]))
    _check(_lib().mm2d_k_maxwellian_field_2d(nx, ny, v1.shape[0], v2.shape[0], _p(rho), _p(u1),
                                             _p(u2), _p(T), _p(v1), _p(v2), _p(M), _stream()))
    res = _host(M)
    if out is None:
        return res
    out[...] = res
    return out


def project_field_2d(F, M, rho, u1, u2, T, v1, v2, dv):
    F, M, rho, u1, u2, T, v1, v2 = (_dev(a) for a in (F, M, rho, u1, u2, T, v1, v2))
    nx, ny, nv1, nv2 = F.shape
    out = _out(F.shape)
    _check(_lib().mm2d_k_project_field_2d(nx, ny, nv1, nv2, _p(F), _p(M), _p(rho), _p(u1), _p(u2),
                                          _p(T), _p(v1), _p(v2), C.c_double(dv), _p(out),
                                          _stream()))
    return _host(out)


def transport_stage_2d(G_ext, M, rho, u1, u2, T, v1, v2, d, dt, axis, out=None):
    G_ext, M, rho, u1, u2, T, v1, v2 = (_dev(a) for a in (G_ext, M, rho, u1, u2, T, v1, v2))
    nx, ny = rho.shape
    nv1, nv2 = v1.shape[0], v2.shape[0]
    o = _out((nx, ny, nv1, nv2))
    _check(_lib().mm2d_k_transport_stage_2d(nx, ny, nv1, nv2, _p(G_ext), _p(M), _p(rho), _p(u1),
                                            _p(u2), _p(T), _p(v1), _p(v2), C.c_double(d),
                                            C.c_double(dt), int(axis), _p(o), _stream()))
    res = _host(o)
    if out is None:
        return res
    out[...] = res
    return out


def ghat_2d(M, rho, u1, u2, T, s11, s12, gT1, gT2, tau, v1, v2, out=None):
    args = [_dev(a) for a in (M, rho, u1, u2, T, s11, s12, gT1, gT2, tau, v1, v2)]
    nx, ny, nv1, nv2 = args[0].shape
    o = _out((nx, ny, nv1, nv2))
    _check(_lib().mm2d_k_ghat_2d(nx, ny, nv1, nv2, *(_p(a) for a in args), _p(o), _stream()))
    res = _host(o)
    if out is None:
        return res
    out[...] = res
    return out


def add_gaussian_term_2d(Ghat, M, rho, u1, u2, m11, m12, m22, eps, v1, v2):
    """In place on Ghat (as the reference kernel); also returns it."""
    g = _dev(Ghat)
    rest = [_dev(a) for a in (M, rho, u1, u2, m11, m12, m22)]
    v1d, v2d = _dev(v1), _dev(v2)
    nx, ny, nv1, nv2 = g.shape
    _check(_lib().mm2d_k_add_gaussian_term_2d(nx, ny, nv1, nv2, _p(g), *(_p(a) for a in rest),
                                              C.c_double(eps), _p(v1d), _p(v2d), _stream()))
    res = _host(g)
    if isinstance(Ghat, np.ndarray):
        Ghat[...] = res
        return Ghat
    return res


def add_lowrank_4d(out, coeffs, shapes):
    """out += sum_m coeffs[m] x shapes[m], in place; also returns out."""
    o = _dev(out)
    c, s = _dev(coeffs), _dev(shapes)
    nx, ny, nv1, nv2 = o.shape
    _check(_lib().mm2d_k_add_lowrank_4d(nx, ny, nv1, nv2, _p(o), int(c.shape[0]), _p(c), _p(s),
                                        _stream()))
    res = _host(o)
    if isinstance(out, np.ndarray):
        out[...] = res
        return out
    return res


def relax_2d(G, Ghat, tau, dt, eps, out=None):
    G, Ghat, tau = _dev(G), _dev(Ghat), _dev(tau)
    nx, ny, nv1, nv2 = G.shape
    o = _out(G.shape)
    _check(_lib().mm2d_k_relax_2d(nx, ny, nv1, nv2, _p(G), _p(Ghat), _p(tau), C.c_double(dt),
                                  C.c_double(eps), _p(o), _stream()))
    res = _host(o)
    if out is None:
        return res
    out[...] = res
    return out


def heat_tensor_2d(G, u1, u2, v1, v2, dv, eps):
    G, u1, u2, v1, v2 = (_dev(a) for a in (G, u1, u2, v1, v2))
    nx, ny, nv1, nv2 = G.shape
    H = _out((4, nx, ny))
    _check(_lib().mm2d_k_heat_tensor_2d(nx, ny, nv1, nv2, _p(G), _p(u1), _p(u2), _p(v1), _p(v2),
                                        C.c_double(dv), C.c_double(eps), _p(H), _stream()))
    h = _host(H)
    return h[0], h[1], h[2], h[3]


__all__ = ["backend_name", "upwind_z_1d", "project_field_1d", "maxwellian_field_2d",
           "project_field_2d", "transport_stage_2d", "ghat_2d", "add_gaussian_term_2d",
           "add_lowrank_4d", "relax_2d", "heat_tensor_2d"]

"""ctypes binding of libmm2d.so, the C ABI declared in include/mm2d.h.

There is no fallback: if the library is missing or fails to load, importing
the device path raises ``NativeLibraryError``.  ``build()`` compiles it with
nvcc for sm_100a (csrc/Makefile).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

from .errors import NativeLibraryError

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libmm2d.so"
CSRC = PKG_DIR / "csrc"

OK, ERR_CONFIG, ERR_STATE, ERR_INTERNAL = 0, 2, 3, 5
STATE_DENSITY, STATE_PRESSURE, STATE_MODIFIED, STATE_TEMPERATURE = 1, 2, 3, 4
STATE_MESSAGES = {
    STATE_DENSITY: "non-positive density",
    STATE_TEMPERATURE: "non-positive temperature",
    STATE_PRESSURE: "pressure tensor is not positive definite",
    STATE_MODIFIED: "modified temperature tensor is not positive definite",
}

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class Config(C.Structure):
    """mirror of struct mm2d_config"""
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int),
        ("x_min", C.c_double), ("x_max", C.c_double),
        ("y_min", C.c_double), ("y_max", C.c_double),
        ("nv1", C.c_int), ("nv2", C.c_int),
        ("v1_min", C.c_double), ("v1_max", C.c_double),
        ("v2_min", C.c_double), ("v2_max", C.c_double),
        ("face", C.c_int * 4),
        ("wall_T", C.c_double * 4),
        ("wall_U", C.c_double * 4),
        ("tau_kind", C.c_int),
        ("tau_value", C.c_double),
        ("nu", C.c_double),
        ("eps", C.c_double),
        ("px", C.c_int), ("py", C.c_int), ("rx", C.c_int), ("ry", C.c_int),
        ("device", C.c_int),
    ]


class Config1D(C.Structure):
    """mirror of struct mm1d_config (include/mm1d.h)"""
    _fields_ = [
        ("nx", C.c_int), ("x_min", C.c_double), ("x_max", C.c_double),
        ("nv", C.c_int), ("v_min", C.c_double), ("v_max", C.c_double),
        ("face", C.c_int * 2),
        ("wall_T", C.c_double * 2),
        ("tau_kind", C.c_int),
        ("tau_value", C.c_double),
        ("eps", C.c_double),
        ("device", C.c_int),
    ]


# every exported symbol with its (restype, argtypes); tests check the .so
# exports exactly these names
SIGNATURES = {
    "mm2d_version": (C.c_int, []),
    "mm2d_kernel_version": (C.c_int, []),
    "mm2d_create": (C.c_int, [C.POINTER(Config), C.POINTER(_vp)]),
    "mm2d_destroy": (C.c_int, [_vp]),
    "mm2d_last_error": (C.c_char_p, [_vp]),
    "mm2d_block": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                             C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "mm2d_step": (C.c_int, [_vp, _vp, _vp, C.c_double, _vp, _vp, _vp, C.c_int,
                            _vp, _vp, _vp, _vp]),
    "mm2d_step_phase": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_double, _vp, _vp, _vp, C.c_int,
                                  _vp, _vp, _vp, _vp]),
    "mm2d_alloc_state": (C.c_int, [_vp]),
    "mm2d_upload": (C.c_int, [_vp, _vp, _vp]),
    "mm2d_upload_device": (C.c_int, [_vp, _vp, _vp]),
    "mm2d_attach_state": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "mm2d_current_index": (C.c_int, [_vp]),
    "mm2d_set_stream": (C.c_int, [_vp, _vp]),
    "mm2d_run": (C.c_int, [_vp, C.c_double, C.c_int]),
    "mm2d_download": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mm2d_state_ptrs": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "mm2d_heat_tensor": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "mm2d_check": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                             C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "mm2d_sync": (C.c_int, [_vp]),
    "mm2d_max_abs_diff": (C.c_int, [_vp, _vp, _vp, C.c_longlong, _vp, _vp]),
    "mm2d_halo_info": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp), C.POINTER(_vp),
                                 C.POINTER(C.c_longlong)]),
    "mm2d_halo_pack": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "mm2d_halo_unpack": (C.c_int, [_vp, C.c_int, _vp]),
    "mm2d_halo_peer": (C.c_int, [_vp, C.POINTER(_vp)]),
    "mm2d_enable_peer_access": (C.c_int, [C.c_int, C.c_int]),
    "mm2d_ipc_alloc": (C.c_int, [C.c_longlong, C.POINTER(_vp), C.c_char_p]),
    "mm2d_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "mm2d_ipc_close": (C.c_int, [_vp]),
    "mm2d_ipc_free": (C.c_int, [_vp]),
    "mm2d_k_maxwellian_field_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 7 + [_vp]),
    "mm2d_k_project_field_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 8 + [C.c_double, _vp, _vp]),
    "mm2d_k_transport_stage_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 8 +
                                  [C.c_double, C.c_double, C.c_int, _vp, _vp]),
    "mm2d_k_ghat_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 12 + [_vp, _vp]),
    "mm2d_k_add_gaussian_term_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 8 +
                                    [C.c_double, _vp, _vp, _vp]),
    "mm2d_k_add_lowrank_4d": (C.c_int, [C.c_int] * 4 + [_vp, C.c_int, _vp, _vp, _vp]),
    "mm2d_k_relax_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 3 + [C.c_double, C.c_double, _vp, _vp]),
    "mm2d_k_heat_tensor_2d": (C.c_int, [C.c_int] * 4 + [_vp] * 5 + [C.c_double, C.c_double,
                                                                     _vp, _vp]),
    "mm2d_k_upwind_z_1d": (C.c_int, [C.c_int, C.c_int, _vp, _vp, C.c_double, _vp, _vp]),
    "mm2d_k_project_field_1d": (C.c_int, [C.c_int, C.c_int] + [_vp] * 6 +
                                [C.c_double, _vp, _vp]),
    "mm2d_time_kernels": (C.c_int, [_vp, C.c_double, C.c_int, _dp]),
    "mm2d_launch_count": (C.c_longlong, []),
    "mm1d_create": (C.c_int, [C.POINTER(Config1D), C.POINTER(_vp)]),
    "mm1d_destroy": (C.c_int, [_vp]),
    "mm1d_last_error": (C.c_char_p, [_vp]),
    "mm1d_step": (C.c_int, [_vp, _vp, _vp, C.c_double, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mm1d_upload": (C.c_int, [_vp, _vp, _vp]),
    "mm1d_run": (C.c_int, [_vp, C.c_double, C.c_int]),
    "mm1d_download": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mm1d_resident": (C.c_int, [_vp]),
    "mm1d_check": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                             C.POINTER(C.c_double)]),
    "mm2d_reset_launch_count": (None, []),
}

_lib = None


def build(force: bool = False) -> Path:
    """Compile libmm2d.so in-tree (nvcc, -gencode arch=compute_100a,code=sm_100a)."""
    if force or not LIB_PATH.exists():
        subprocess.run(["make", "-C", str(CSRC)], check=True)
    else:
        subprocess.run(["make", "-C", str(CSRC)], check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


def load():
    """Load libmm2d.so and declare its prototypes (raises if unavailable)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("MM2D_LIBRARY", str(LIB_PATH))
    if not Path(path).exists():
        raise NativeLibraryError(
            f"{path} is missing; build it with `make -C {CSRC}` "
            "(the device path has no CPU fallback)")
    try:
        lib = C.CDLL(path)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error(ctx) -> str:
    msg = load().mm2d_last_error(ctx)
    return msg.decode() if msg else ""

"""The C-ABI library loads and exports every symbol include/mm2d.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import re
import subprocess

from conftest import ROOT


def header_symbols():
    syms = set()
    for h in ("mm2d.h", "mm1d.h"):
        text = (ROOT / "include" / h).read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(mm[12]d_\w+)\s*\(", text))
    return sorted(syms)


def test_header_declares_the_boundary():
    syms = header_symbols()
    for required in ("mm2d_create", "mm2d_step", "mm2d_run", "mm2d_check",
                     "mm2d_k_transport_stage_2d", "mm2d_k_heat_tensor_2d"):
        assert required in syms
    assert len([s for s in syms if s.startswith("mm2d_k_")]) == 10
    for required in ("mm1d_create", "mm1d_step", "mm1d_run", "mm1d_check"):
        assert required in syms


def test_library_exports_every_header_symbol():
    from paper_2509_21832_b200 import _native
    _native.build()
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares exactly the header's functions
    assert sorted(_native.SIGNATURES) == header_symbols()


def test_library_is_sm100a():
    from paper_2509_21832_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_callable_without_gpu():
    from paper_2509_21832_b200 import _native
    lib = _native.load()
    assert lib.mm2d_version() >= 1

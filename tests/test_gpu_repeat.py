"""Race and determinism probes for the fused kernels (compute-sanitizer is
closed on the GPU pool: profiles/r02_compute_sanitizer_closed.log).

A read of shared or tensor memory before its producer finished (a missing
barrier, an mbarrier phase slip, a table slot reused too early) makes the
result depend on CTA timing.  These tests change the timing and demand
bit-identical results:

  * the same step twice in one process;
  * the same step under different band layouts of the 32 x 32 kernel
    (MM2D_LY / MM2D_BANDS: different CTA counts, band ends and co-resident
    CTA mixes), each in a fresh process;
  * the debug build (MM2D_DEBUG_CHECKS, device-side bounds checks on every
    shared / tensor / global index the kernels compute) on the same inputs.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import bench, paper_2509_21832_b200 as mm
cfg = bench.make_workload({name!r}, n={n})
st = mm.State2D(0.0, cfg["initial"](0, {n}, 0, {n}), np.zeros(({n}, {n}, 32, 32)))
for _ in range({steps}):
    st = mm.step_2d(st, cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"], cfg["dt"])
np.savez({out!r}, Q=st.Q, G=st.G, H=st.H_step.cpu().numpy())
"""


def _run(tmp_path, tag, env_extra, name="c5", n=64, steps=3):
    out = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ, **env_extra)
    code = SCRIPT.format(root=str(ROOT), name=name, n=n, steps=steps, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("name", ["c5", "c4", "c4s", "c3"])
def test_band_layouts_give_identical_bits(gpu, tmp_path, name):
    ref = _run(tmp_path, "default", {}, name=name)
    for tag, env in [("ly8", {"MM2D_LY": "8"}), ("ly13", {"MM2D_LY": "13"}),
                     ("ly64", {"MM2D_LY": "64"}), ("bands", {"MM2D_BANDS": "5,24,35"}),
                     ("again", {})]:
        d = _run(tmp_path, tag, env, name=name)
        for k in ("Q", "G", "H"):
            assert np.array_equal(d[k], ref[k]), (name, tag, k)


def test_debug_build_checks_pass_and_match(gpu, tmp_path):
    dbg = ROOT / "paper_2509_21832_b200" / "libmm2d_dbg.so"
    if not dbg.exists():
        pytest.skip("libmm2d_dbg.so not built (make EXTRA=-DMM2D_DEBUG_CHECKS=1 ...)")
    for name in ("c5", "c4", "c4s"):
        ref = _run(tmp_path, f"rel_{name}", {}, name=name, n=24)
        d = _run(tmp_path, f"dbg_{name}", {"MM2D_LIBRARY": str(dbg)}, name=name, n=24)
        for k in ("Q", "G", "H"):
            assert np.array_equal(d[k], ref[k]), (name, k)

"""Small runs of every production kernel for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per call):

  k_micro32<4,false>  C5 generator, 8 x 8 cells, periodic (+ the split
                      interior/perimeter launches of a 2 x 2 block grid)
  k_micro32<4,true>   specular box, 8 x 8 cells
  k_wall_ghat         diffuse-wall box, 8 x 8 cells
  k_prep_tiled, k_macro_x, k_macro_y   every step above
  k_micro (generic)   8 x 8 cells, 12 x 10 velocities
  k1_micro/k1_macro   1D Sod, 64 cells, single steps
  k1_resident         1D Sod, 64 cells, a 20-step cluster-resident run

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_21832_b200 as mm  # noqa: E402
from paper_2509_21832_b200.parallel import run_parallel_2d  # noqa: E402


def steps(cfg, n, Q0=None, G0=None):
    nx, ny = cfg["nx"], cfg["ny"]
    Q0 = cfg["initial"](0, nx, 0, ny) if Q0 is None else Q0
    G0 = np.zeros((nx, ny) + tuple(a.n for a in cfg["mesh"].velocity)) if G0 is None else G0
    st = mm.State2D(0.0, Q0, G0)
    for _ in range(n):
        st = mm.step_2d(st, cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"], cfg["dt"])
    return st.Q, st.G


def main():
    torch.cuda.set_device(0)
    c5 = bench.make_workload("c5", n=8)
    Q, G = steps(c5, 2)
    assert np.isfinite(Q).all() and np.isfinite(G).all()
    Qp, _, _, _ = run_parallel_2d(c5["mesh"], c5["bc"], c5["eps"], c5["model"],
                                  c5["initial"](0, 8, 0, 8), np.zeros((8, 8, 32, 32)), c5["dt"], 2,
                                  grid=(2, 2), graph=False)
    assert np.isfinite(Qp).all()
    spec = bench.make_workload("c4s", n=8)
    Q, G = steps(spec, 2)
    assert np.isfinite(Q).all()
    walls = bench.make_workload("c4", n=8)
    Q, G = steps(walls, 2)
    assert np.isfinite(Q).all()
    # generic kernel: odd velocity counts
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, 8), mm.Axis(0.0, 1.0, 8)),
                        velocity=(mm.Axis(-6.0, 6.0, 12), mm.Axis(-6.0, 6.0, 10)))
    gen = dict(c5, mesh=mesh, nx=8, ny=8)
    Q, G = steps(gen, 2, Q0=c5["initial"](0, 8, 0, 8), G0=np.zeros((8, 8, 12, 10)))
    assert np.isfinite(Q).all()
    # 1D: single steps and a resident run
    mesh1 = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, 64),), velocity=(mm.Axis(-8.0, 8.0, 64),))
    bc1 = mm.BoundarySpec1D(mm.EXTRAPOLATE, mm.EXTRAPOLATE)
    model1 = mm.CollisionModel("hard_sphere_1d")
    x = (np.arange(64) + 0.5) / 64
    rho = np.where(x < 0.5, 1.0, 0.125)
    T = np.where(x < 0.5, 1.0, 0.8)
    st1 = mm.State1D(0.0, mm.conserved_1d(rho, 0 * x, T), np.zeros((64, 64)))
    for _ in range(2):
        st1 = mm.step_1d(st1, mesh1, bc1, 1e-2, model1, 1e-3)
    assert np.isfinite(st1.Q).all()
    st1, _ = mm.run_1d(mesh1, bc1, 1e-2, model1, rho, 0 * x, T, np.zeros((64, 64)), 0.004, 0.4)
    assert np.isfinite(st1.Q).all()
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()

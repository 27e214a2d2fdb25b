"""Time the config-1 run (Sod, 256 x 64, 512 steps) on the GPU: the
cluster-resident single launch vs the graph replay of the two-kernel step.
mm1d_run is asynchronous on the context stream; mm1d_download(NULL...) is
the synchronisation point, so run+sync is timed for several step counts and
the per-step cost is the slope (fixed costs cancel)."""

import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200.solver1d import Solver1D
    from paper_2509_21832_b200 import (EXTRAPOLATE, Axis, BoundarySpec1D, CollisionModel,
                                       PhaseMesh, cell_centers)
    mesh = PhaseMesh(space=(Axis(0.0, 1.0, 256),), velocity=(Axis(-8.0, 8.0, 64),))
    bc = BoundarySpec1D(EXTRAPOLATE, EXTRAPOLATE)
    x = cell_centers(mesh.space[0])
    rho = np.where(x < 0.5, 1.0, 0.125)
    T = np.where(x < 0.5, 1.0, 0.8)
    Q0 = np.ascontiguousarray(mm.conserved_1d(rho, 0 * rho, T))
    G0 = np.zeros((256, 64))
    plan = mm.plan_time(0.1, 0.4, mesh)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    modes = sys.argv[1:] or ["resident", "graph"]
    for mode in modes:
        if mode == "graph":
            os.environ["MM1D_NO_RESIDENT"] = "1"
        s = Solver1D(mesh, bc, 1e-2, CollisionModel("hard_sphere_1d"))
        lib, ctx = s.lib, s.ctx
        res = {}
        for n in (1, 64, 512, 2048):
            best = 1e9
            for rep in range(6):
                lib.mm1d_upload(ctx, p(Q0), p(G0))
                t0 = time.perf_counter()
                lib.mm1d_run(ctx, C.c_double(plan.dt), n)
                lib.mm1d_download(ctx, None, None, None)
                dt = time.perf_counter() - t0
                if rep:
                    best = min(best, dt)
            res[n] = best
        slope = (res[2048] - res[64]) / (2048 - 64)
        print(f"{mode}: resident={s.resident} " +
              " ".join(f"n={n}:{t * 1e3:.3f}ms" for n, t in res.items()) +
              f"  -> {slope * 1e6:.2f} us/step, 512-step run {res[512] * 1e3:.3f} ms = "
              f"{256 * 64 * 512 / res[512]:.3e} node-updates/s")
        s.close()


if __name__ == "__main__":
    main()

"""Micro-kernel time per node against the grid shape (tail and wave
effects): periodic density-wave problems of different (nx, ny), with the
library's own band choice (MM2D_VERBOSE=1 prints it).

    python tools/wave_probe.py [nx,ny ...]
"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200.solver import Solver2D
    shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [
        (256, 256), (256, 1024), (1024, 256), (512, 512), (1024, 1024), (296, 256)]
    for nx, ny in shapes:
        mesh = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, nx), mm.Axis(0.0, 1.0, ny)),
                            velocity=(mm.Axis(-7.0, 7.0, 32), mm.Axis(-7.0, 7.0, 32)))
        bc = mm.BoundarySpec2D(mm.PERIODIC, mm.PERIODIC, mm.PERIODIC, mm.PERIODIC)
        model = mm.CollisionModel("esbgk_2d", nu=-0.5)
        s = Solver2D(mesh, bc, 0.1, model)
        x = (np.arange(nx) + 0.5) / nx
        rho = 1.0 + 0.2 * np.sin(2 * np.pi * x)[:, None] * np.ones((1, ny))
        z = np.zeros_like(rho)
        Q = torch.from_numpy(mm.conserved_2d(rho, z, z, np.ones_like(rho), z, np.ones_like(rho))).cuda()
        G = torch.zeros((nx, ny, 32, 32), dtype=torch.float64, device="cuda")
        Qb, Gb = torch.empty_like(Q), torch.empty_like(G)
        H = torch.empty((4, nx, ny), dtype=torch.float64, device="cuda")
        p = lambda t: C.c_void_p(t.data_ptr())
        s.lib.mm2d_attach_state(s.ctx, p(Q), p(G), p(Qb), p(Gb), p(H))
        ms = (C.c_double * 7)()
        dt = 0.4 * (1.0 / nx) / 7.0
        s.lib.mm2d_time_kernels(s.ctx, C.c_double(dt), 3, ms)
        s.lib.mm2d_time_kernels(s.ctx, C.c_double(dt), 10, ms)
        ns = ms[2] * 1e6 / (nx * ny * 1024)
        print(f"{nx}x{ny}: micro {ms[2]:.4f} ms  {ns * 1000:.3f} ps/node", flush=True)
        s.close()


if __name__ == "__main__":
    main()

"""Micro-kernel time per node against the CTA-wave count (tail cost):
periodic density-wave problems of different (nx, ny), ly = 48 bands.

    python tools/wave_probe.py
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
    for nx, ny in [(222, 288), (256, 256), (259, 288), (296, 288), (148, 480), (444, 96)]:
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
        ctas = nx * ((ny + 47) // 48)
        ns = ms[2] * 1e6 / (nx * ny * 1024)
        print(f"{nx}x{ny}: {ctas} CTAs = {ctas / 444:.2f} waves  micro {ms[2]:.4f} ms  "
              f"{ns * 1000:.2f} ps/node")
        s.close()


if __name__ == "__main__":
    main()

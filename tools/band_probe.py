"""Micro-kernel time against the band height on one grid shape (periodic
x-wave state; MM2D_LY is read when the context is created).

    python tools/band_probe.py NX NY LY[,LY...] [auto]
"""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200.solver import Solver2D
    nx, ny = int(sys.argv[1]), int(sys.argv[2])
    lys = [int(v) for v in sys.argv[3].split(",")] + ([0] if "auto" in sys.argv[4:] else [])
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, nx), mm.Axis(0.0, 1.0, ny)),
                        velocity=(mm.Axis(-7.0, 7.0, 32), mm.Axis(-7.0, 7.0, 32)))
    bc = mm.BoundarySpec2D(mm.PERIODIC, mm.PERIODIC, mm.PERIODIC, mm.PERIODIC)
    model = mm.CollisionModel("esbgk_2d", nu=-0.5)
    x = (np.arange(nx) + 0.5) / nx
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * x)[:, None] * np.ones((1, ny))
    z = np.zeros_like(rho)
    Q = torch.from_numpy(mm.conserved_2d(rho, z, z, np.ones_like(rho), z, np.ones_like(rho))).cuda()
    G = torch.zeros((nx, ny, 32, 32), dtype=torch.float64, device="cuda")
    Qb, Gb = torch.empty_like(Q), torch.empty_like(G)
    H = torch.empty((4, nx, ny), dtype=torch.float64, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    dt = 0.4 * (1.0 / max(nx, ny)) / 7.0
    for rnd in range(2):
        for ly in lys:
            if ly:
                os.environ["MM2D_LY"] = str(ly)
            else:
                os.environ.pop("MM2D_LY", None)
            s = Solver2D(mesh, bc, 0.1, model)
            s.lib.mm2d_attach_state(s.ctx, p(Q), p(G), p(Qb), p(Gb), p(H))
            ms = (C.c_double * 7)()
            s.lib.mm2d_time_kernels(s.ctx, C.c_double(dt), 2, ms)
            s.lib.mm2d_time_kernels(s.ctx, C.c_double(dt), 5, ms)
            print(f"{nx}x{ny} ly {ly or 'auto'}: micro {ms[2]:.4f} ms  "
                  f"{ms[2] * 1e9 / (nx * ny * 1024):.3f} ps/node", flush=True)
            s.close()


if __name__ == "__main__":
    main()

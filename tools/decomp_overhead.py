"""Device cost of the block decomposition on ONE GPU: the same periodic
problem advanced serially and as a block grid held by one process (peer-form
and packed G halos, CUDA-graph replay), seconds per step from
run_parallel_2d's own device-synchronised timer.  No NVLink is involved: this
isolates what the decomposition itself adds (Q / H ring packs and copies,
extra launches, the perimeter CTAs' halo reads).

    python tools/decomp_overhead.py [--nx 512 --ny 1024 --steps 20]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=512)
    ap.add_argument("--ny", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--big", action="store_true",
                    help="only the 2x2 grid (for blocks of the C5 x 8 GPU size: --nx 1024 --ny 2048)")
    args = ap.parse_args()
    import bench
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200.parallel import run_parallel_2d
    nx, ny = args.nx, args.ny
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, nx), mm.Axis(0.0, ny / nx, ny)),
                        velocity=(mm.Axis(-7.0, 7.0, 32), mm.Axis(-7.0, 7.0, 32)))
    bc = mm.BoundarySpec2D(*(mm.PERIODIC,) * 4)
    model = mm.CollisionModel("esbgk_2d", nu=-0.5)
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / nx
    X, Y = np.meshgrid(x, y, indexing="ij")
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.cos(np.pi * Y)
    Q0 = mm.conserved_2d(rho, 0.1 * np.cos(2 * np.pi * X), 0.0 * X, 1.0 + 0 * X, 0 * X, 1.0 + 0 * X)
    G0 = np.zeros((nx, ny, 32, 32))
    dt = 0.4 * (1.0 / nx) / 7.0
    base = None
    grids = [(1, 1), (2, 2)] if args.big else [(1, 1), (2, 2), (4, 2)]
    for grid, halo in [(g, h) for g in grids for h in (("peer",) if g == (1, 1) else
                                                       ("peer", "packed"))]:
        best = 1e9
        for _ in range(2):
            Q, G, _, sec = run_parallel_2d(mesh, bc, 0.01, model, Q0, G0, dt, args.steps, grid=grid,
                                           halo=halo)
            best = min(best, sec / args.steps)
        if base is None:
            base, Qs = best, Q
        same = bool(np.array_equal(Q, Qs))
        print(f"grid {grid[0]}x{grid[1]} halo {halo:6s}: {1e3 * best:8.3f} ms/step "
              f"({best / base:5.3f} x serial), bitwise serial: {same}", flush=True)


if __name__ == "__main__":
    main()

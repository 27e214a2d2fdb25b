"""Host-side issue cost of one decomposed step (step_blocks) against its
device time, on one GPU with the loopback transport: a 1-block "grid" with
periodic halo faces exchanged with itself, so every protocol call of the
multi-rank step runs (packs, exchanges, split phases, unpacks).

    python tools/host_issue_probe.py [n_cells_per_side] [steps]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200.parallel import (BlockStepper, LoopbackExchange, make_plans,
                                                step_blocks)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    for grid in [(2, 1), (2, 2)]:
        nx, ny = n * grid[0], n * grid[1]
        mesh = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, nx), mm.Axis(0.0, 1.0, ny)),
                            velocity=(mm.Axis(-7.0, 7.0, 32), mm.Axis(-7.0, 7.0, 32)))
        bc = mm.BoundarySpec2D(mm.PERIODIC, mm.PERIODIC, mm.PERIODIC, mm.PERIODIC)
        model = mm.CollisionModel("esbgk_2d", nu=-0.5)
        plans = make_plans(nx, ny, grid, bc)
        dev = torch.device("cuda", 0)
        blocks, states = [], []
        for p in plans:
            b = BlockStepper(mesh, bc, 0.1, model, grid, p, dev)
            blocks.append(b)
            x = (np.arange(p.i0, p.i1) + 0.5) / nx
            rho = 1.0 + 0.2 * np.sin(2 * np.pi * x)[:, None] * np.ones((1, p.shape[1]))
            z = np.zeros_like(rho)
            Q = torch.from_numpy(mm.conserved_2d(rho, z + 0.5, z + 0.5, np.ones_like(rho), z,
                                                 np.ones_like(rho))).to(dev)
            G = torch.zeros(p.shape + (32, 32), dtype=torch.float64, device=dev)
            states.append([Q, G, torch.empty_like(Q), torch.empty_like(G),
                           torch.empty((4,) + p.shape, dtype=torch.float64, device=dev)])
        ex = LoopbackExchange(plans, [b.bufs for b in blocks])
        dt = 0.4 / max(nx, ny) / 7.0

        def run(k):
            for _ in range(k):
                step_blocks(blocks, ex, states, dt)
                for st in states:
                    st[0], st[2] = st[2], st[0]
                    st[1], st[3] = st[3], st[1]

        run(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        run(steps)
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1) / steps
        host_ms = (h1 - h0) * 1e3 / steps
        nb = len(blocks)
        print(f"grid {grid}: {nb} blocks of {n}x{n}: device {dev_ms:.3f} ms/step "
              f"({dev_ms / nb:.3f} per block), host issue {host_ms:.3f} ms/step "
              f"({host_ms / nb:.3f} per block)", flush=True)
        for b in blocks:
            b.solver.check()
            b.solver.close()


if __name__ == "__main__":
    main()

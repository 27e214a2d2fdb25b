"""Step time of a bench workload against explicit k_micro32 band layouts
(MM2D_BANDS, read when the context is created): the bench's own timed loop
(Solver2D.run graph replays, CUDA events), alternating rounds.

    python tools/bands_bench.py CONFIG "LAYOUT;LAYOUT;..." [steps] [nx ny]
    LAYOUT = comma-separated band heights, or "auto" for the library's choice
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_21832_b200.solver import Solver2D  # noqa: E402


def main():
    layouts = sys.argv[2].split(";")
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    n = None
    cfg = bench.make_workload(sys.argv[1])
    if len(sys.argv) > 5:   # a block of another shape (same dx, dt): the multi-GPU block sizes
        import paper_2509_21832_b200 as mm
        nx, ny = int(sys.argv[4]), int(sys.argv[5])
        dx = cfg["mesh"].space[0].spacing
        cfg = dict(cfg, nx=nx, ny=ny,
                   mesh=mm.PhaseMesh(space=(mm.Axis(0.0, nx * dx, nx), mm.Axis(0.0, ny * dx, ny)),
                                     velocity=cfg["mesh"].velocity))
        full = cfg["initial"]
        cfg["initial"] = lambda i0, i1, j0, j1: full(i0, i1, j0, j1)
    Q0 = torch.from_numpy(cfg["initial"](0, cfg["nx"], 0, cfg["ny"])).cuda()
    Q = Q0.clone()
    G = torch.zeros((cfg["nx"], cfg["ny"], 32, 32), dtype=torch.float64, device="cuda")
    for rnd in range(3):
        for lay in layouts:
            if lay == "auto":
                os.environ.pop("MM2D_BANDS", None)
            else:
                os.environ["MM2D_BANDS"] = lay
            s = Solver2D(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"])
            Qb, Gb = s.empty_state()
            H = torch.empty((4, cfg["nx"], cfg["ny"]), dtype=torch.float64, device="cuda")
            Q.copy_(Q0)
            G.zero_()
            s.run(Q, G, cfg["dt"], 3, H_out=H, Q_b=Qb, G_b=Gb)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.run(Q, G, cfg["dt"], steps, H_out=H, Q_b=Qb, G_b=Gb)
            e1.record()
            torch.cuda.synchronize()
            s.check()
            print(f"{sys.argv[1]} {cfg['nx']}x{cfg['ny']} bands {lay}: "
                  f"{e0.elapsed_time(e1) / steps:.4f} ms/step", flush=True)
            del Qb, Gb, H
            s.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

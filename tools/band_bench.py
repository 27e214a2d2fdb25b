"""Step time of a bench workload against the k_micro32 band height: the
bench's own timed loop (Solver2D.run graph replays, CUDA events), two
alternating rounds.  MM2D_LY is read when the context is created.

    python tools/band_bench.py CONFIG LY[,LY...] [steps]      (LY 0 = library choice)
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
    cfg = bench.make_workload(sys.argv[1])
    lys = [int(v) for v in sys.argv[2].split(",")]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    Q0 = torch.from_numpy(cfg["initial"](0, cfg["nx"], 0, cfg["ny"])).cuda()
    Q = Q0.clone()
    G = torch.zeros((cfg["nx"], cfg["ny"], 32, 32), dtype=torch.float64, device="cuda")
    for rnd in range(2):
        for ly in lys:
            if ly:
                os.environ["MM2D_LY"] = str(ly)
            else:
                os.environ.pop("MM2D_LY", None)
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
            print(f"{sys.argv[1]} ly {ly or 'auto'}: {e0.elapsed_time(e1) / steps:.4f} ms/step",
                  flush=True)
            del Qb, Gb, H
            s.close()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

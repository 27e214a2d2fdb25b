"""Run a few plain (non-graph) steps of a benchmark workload, for ncu.

    python tools/profile_step.py [--config c2] [--steps 4]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_21832_b200.solver import Solver2D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--n", type=int, default=None, help="cells per axis (default: the config's)")
    ap.add_argument("--run", action="store_true",
                    help="ping-pong through Solver2D.run (two state buffers, no allocations "
                         "per step: the C5 state is 32 GiB per copy)")
    args = ap.parse_args()
    cfg = bench.make_workload(args.config, n=args.n)
    s = Solver2D(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"])
    Q = torch.from_numpy(cfg["initial"](0, cfg["nx"], 0, cfg["ny"])).cuda()
    G = torch.zeros((cfg["nx"], cfg["ny"], 32, 32), dtype=torch.float64, device="cuda")
    if args.run:
        Qb, Gb = s.empty_state()
        Q, G = s.run(Q, G, cfg["dt"], args.steps, Q_b=Qb, G_b=Gb)
    else:
        for _ in range(args.steps):
            Q, G, H = s.step(Q, G, cfg["dt"])
    torch.cuda.synchronize()
    s.check()
    print("ok", float(Q[..., 0].sum()))


if __name__ == "__main__":
    main()

"""Functional check of the one-process-per-GPU decomposed step: under
torchrun (gloo, every rank may share one GPU), advance a small periodic /
walled problem with the block grid spread over the ranks, gather the blocks on
rank 0 and compare bit for bit with the serial step_2d.

    python -m torch.distributed.run --nproc-per-node 4 tools/multirank_check.py \
        --grid 2 2 --halo peer

--halo peer maps the neighbours' G buffers with CUDA IPC and reads the ghost
cells in place (IpcPeers); --halo packed sends the packed G ring.  No kernel
waits on another rank: the exchanges are host-staged (DistExchange staged)."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, nargs=2, default=[2, 1])
    ap.add_argument("--halo", default="peer", choices=["peer", "packed"])
    ap.add_argument("--faces", default="periodic", choices=["periodic", "cavity", "mixed"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nv", type=int, default=32)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200.parallel import (BlockStepper, DistExchange, IpcPeers, make_plans,
                                                step_blocks)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    px, py = args.grid
    assert px * py == world
    nx, ny, nv = 12 * px, 20 * py, args.nv
    w = mm.WallSpec(1.0)
    faces = {"periodic": (mm.PERIODIC,) * 4, "cavity": (w, w, w, mm.WallSpec(1.0, 0.16)),
             "mixed": (mm.EXTRAPOLATE, mm.EXTRAPOLATE, mm.PERIODIC, mm.PERIODIC)}[args.faces]
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, 1.0, nx), mm.Axis(0.0, 1.0, ny)),
                        velocity=(mm.Axis(-5.0, 5.0, nv), mm.Axis(-5.0, 5.0, nv)))
    bc = mm.BoundarySpec2D(*faces)
    model = mm.CollisionModel("esbgk_2d", nu=-0.5)
    x = (np.arange(nx) + 0.5) / nx
    y = (np.arange(ny) + 0.5) / ny
    X, Y = np.meshgrid(x, y, indexing="ij")
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)
    T = 1.0 + 0.1 * np.cos(2 * np.pi * X)
    Q0 = mm.conserved_2d(rho, 0.02 * np.cos(2 * np.pi * Y), -0.03 * np.sin(2 * np.pi * X), T,
                         0.02 * np.sin(2 * np.pi * (X + Y)), T)
    G0 = 0.01 * np.random.default_rng(7).standard_normal((nx, ny, nv, nv))
    dt, eps = 0.3 * min(1.0 / nx, 1.0 / ny) / 5.0, 0.08
    plan = make_plans(nx, ny, (px, py), bc)[rank]
    blk = BlockStepper(mesh, bc, eps, model, (px, py), plan, torch.device("cuda", dev))
    exch = DistExchange(plan, blk.bufs, staged=True)
    bx, by = plan.shape
    peers = None
    if args.halo == "peer":
        peers = IpcPeers(blk.solver, plan, (bx, by, nv, nv))
        assert peers.failed is None, peers.failed
        G, Gb = peers.tensors
        G.copy_(torch.from_numpy(np.ascontiguousarray(G0[plan.i0:plan.i1, plan.j0:plan.j1])))
    else:
        G = torch.from_numpy(np.ascontiguousarray(G0[plan.i0:plan.i1, plan.j0:plan.j1])).cuda()
        Gb = torch.empty_like(G)
    Q = torch.from_numpy(np.ascontiguousarray(Q0[plan.i0:plan.i1, plan.j0:plan.j1])).cuda()
    st = [Q, G, torch.empty_like(Q), Gb, torch.empty((4, bx, by), dtype=torch.float64,
                                                     device="cuda")]
    dist.barrier()
    par = 0
    for _ in range(args.steps):
        step_blocks([blk], exch, [st], dt,
                    peers=[peers.views(par)] if peers is not None else None)
        st[0], st[2] = st[2], st[0]
        st[1], st[3] = st[3], st[1]
        par ^= 1
    torch.cuda.synchronize()
    blk.solver.check()
    parts = [None] * world if rank == 0 else None
    dist.gather_object((plan.i0, plan.i1, plan.j0, plan.j1, st[0].cpu().numpy(),
                        st[1].cpu().numpy()), parts, dst=0)
    ok = True
    if rank == 0:
        Q, G = np.empty_like(Q0), np.empty_like(G0)
        for i0, i1, j0, j1, q, g in parts:
            Q[i0:i1, j0:j1], G[i0:i1, j0:j1] = q, g
        s = mm.State2D(0.0, Q0, G0)
        for _ in range(args.steps):
            s = mm.step_2d(s, mesh, bc, eps, model, dt)
        ok = bool(np.array_equal(Q, s.Q) and np.array_equal(G, s.G))
        print(f"multirank_check grid {px}x{py} halo {args.halo} faces {args.faces} nv {nv}: "
              + ("BITWISE OK" if ok else f"MISMATCH dQ {np.abs(Q - s.Q).max():.3e} "
                                         f"dG {np.abs(G - s.G).max():.3e}"), flush=True)
    dist.barrier()
    if peers is not None:
        del st, G, Gb
        peers.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

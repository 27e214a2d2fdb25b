#!/usr/bin/env python
"""Benchmark of the micro-macro ES-BGK 2D2V timestep on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c4s|c5|weak]
                  [--impl ours|reference]

A "step" is one full timestep of the hot path (prep -> fused micro kernel ->
macro KFVS/TR-BDF2) over the whole grid.  Default workload at N=1 is
BASELINE.json configs[1] (C2: 256^2 x 32^2 periodic density wave, fp64).
Metric: phase-space node-updates/s = nx*ny*nv1*nv2*K / seconds (device
time, CUDA events, max over ranks).  G is 512 MiB at C2 (> 126 MB L2), so
no L2 flush is needed between steps.

--impl reference times the reference algorithm's CPU path (the C oracle
port of the reference kernels, OpenMP over all host cores) on a bounded
sample of the same workload; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "phase-space node-updates/s (fp64, 2D-2V) and % of B200 HBM roofline"
UNIT = "node-updates/s"


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------

def c5_fields(seed, X, Y):
    """Random smooth macro state, a pure function of (seed, x, y):
    4 Fourier modes with integer k, 1 <= |k| <= 4, random phases."""
    rng = np.random.default_rng(seed)
    ks = []
    while len(ks) < 12:
        k = rng.integers(-4, 5, size=2)
        if 1 <= math.hypot(*k) <= 4:
            ks.append(k)
    ph = rng.uniform(0, 2 * np.pi, 12)

    def psi(m):
        return sum(np.cos(2 * np.pi * (ks[4 * m + q][0] * X + ks[4 * m + q][1] * Y) + ph[4 * m + q])
                   for q in range(4)) / 4.0

    p0, p1, p2 = psi(0), psi(1), psi(2)
    return 1.0 + 0.1 * p0, 0.2 * p1, 0.2 * p2, 1.0 + 0.05 * p0


def make_workload(name, n_gpus=1, px=1, py=1):
    import paper_2509_21832_b200 as mm
    if name == "c2":
        n, v, faces, eps, ic = 256, (-7.0, 7.0), "periodic", 0.1, "wave"
        wl = "C2 smooth periodic density wave 256^2 x 32^2 (BASELINE configs[1])"
        if px * py > 1:
            wl = (f"C2 weak scaling: 256^2 x 32^2 per GPU, periodic wave tiled on "
                  f"{px}x{py} GPUs ({256 * px}x{256 * py} cells)")
        nx, ny = n * px, n * py
        Lx, Ly = float(px), float(py)
    elif name == "c3":
        nx = ny = 512
        v, faces, eps, ic = (-8.0, 8.0), "extrapolate", 1e-2, "riemann"
        wl = "C3 four-quadrant Riemann 512^2 x 32^2 outflow(extrapolate), eps=1e-2"
        Lx = Ly = 1.0
    elif name == "c4":
        nx = ny = 1024
        v, faces, eps, ic = (-8.0, 8.0), "walls", 5e-2, "bump"
        wl = "C4 closed box, diffuse walls, 1024^2 x 32^2, eps=5e-2"
        Lx = Ly = 1.0
    elif name == "c4s":
        nx = ny = 1024
        v, faces, eps, ic = (-8.0, 8.0), "specular", 5e-2, "bump"
        wl = "C4 closed box, specular walls (BASELINE wording), 1024^2 x 32^2, eps=5e-2"
        Lx = Ly = 1.0
    elif name == "c5":
        nx = ny = 2048
        v, faces, eps, ic = (-7.0, 7.0), "periodic", 1e-2, "fourier"
        wl = "C5 strong-scaling 2048^2 x 32^2 periodic random Fourier, eps=1e-2"
        Lx = Ly = 1.0
    elif name in ("weak", "c5w"):
        nx, ny = 1024 * px, 1024 * py
        v, faces, eps, ic = (-7.0, 7.0), "periodic", 1e-2, "fourier"
        wl = f"C5 weak scaling 1024^2 x 32^2 per GPU ({nx}x{ny} total)"
        Lx, Ly = float(px), float(py)
    else:
        raise SystemExit(f"unknown config {name}")
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, Lx, nx), mm.Axis(0.0, Ly, ny)),
                        velocity=(mm.Axis(v[0], v[1], 32), mm.Axis(v[0], v[1], 32)))
    if faces == "periodic":
        bc = mm.BoundarySpec2D(mm.PERIODIC, mm.PERIODIC, mm.PERIODIC, mm.PERIODIC)
    elif faces == "extrapolate":
        bc = mm.BoundarySpec2D(mm.EXTRAPOLATE, mm.EXTRAPOLATE, mm.EXTRAPOLATE, mm.EXTRAPOLATE)
    elif faces == "specular":
        bc = mm.BoundarySpec2D(mm.SPECULAR, mm.SPECULAR, mm.SPECULAR, mm.SPECULAR)
    else:
        w = mm.WallSpec(1.0, 0.0)
        bc = mm.BoundarySpec2D(w, w, w, w)
    model = mm.CollisionModel("esbgk_2d", nu=-0.5)
    vmax = max(abs(v[0]), abs(v[1]))
    dt = 0.4 * min(Lx / nx, Ly / ny) / vmax

    def initial(i0, i1, j0, j1):
        x = (np.arange(i0, i1) + 0.5) * (Lx / nx)
        y = (np.arange(j0, j1) + 0.5) * (Ly / ny)
        X, Y = np.meshgrid(x, y, indexing="ij")
        one = np.ones_like(X)
        if ic == "wave":
            rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)
            u1, u2, T = 0.5 * one, 0.5 * one, one
        elif ic == "riemann":
            north, east = Y >= 0.5, X >= 0.5
            rho = np.where(north, np.where(east, 1.0, 0.5), np.where(east, 0.5, 0.25))
            u1 = np.where(north, np.where(east, 0.0, 0.5), np.where(east, 0.0, 0.5))
            u2 = np.where(north, 0.0, 0.5)
            T = np.where(north, np.where(east, 1.0, 0.8), np.where(east, 0.8, 0.6))
        elif ic == "bump":
            rho = 1.0 + 0.5 * np.exp(-((X - 0.3) ** 2 + (Y - 0.6) ** 2) / 0.01)
            u1, u2, T = 0 * one, 0 * one, one
        else:
            rho, u1, u2, T = c5_fields(0, X, Y)
        return mm.conserved_2d(rho, u1, u2, T, 0 * one, T)

    # the run length each config names (C3: t = 0.1 at this dt)
    run_steps = {"c2": 100, "c3": int(np.ceil(0.1 / dt - 1e-9)), "c4": 200, "c4s": 200}.get(name, 50)
    return dict(name=name, workload=wl, mesh=mesh, bc=bc, eps=eps, model=model, dt=dt,
                initial=initial, nx=nx, ny=ny, V=32 * 32, run_steps=run_steps)


def bytes_per_step(nx, ny, V):
    """Algorithmic bytes of one timestep: read G^n, write
    G^{n+1} (8 B each per node) + read/write Q (2 x 6 x 8 B per cell)."""
    return nx * ny * (16 * V + 96)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = []
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        inwin = [r for r in rows if t0 is None or (t0 <= r[0] <= t1)]
        use = inwin if inwin else rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in use for q in range(4) if r[3][q].lower() == "active"})
        return {"sm_mhz": statistics.median(r[1] for r in use), "sm_max_mhz": max(r[2] for r in use),
                "reasons": reasons, "samples": len(use), "in_timed_window": bool(inwin)}


# ---------------------------------------------------------------------------
# CPU arm (reference algorithm, C oracle port)
# ---------------------------------------------------------------------------

def cpu_sample(cfg, budget_s, threads=None):
    """Time the oracle (C restatement of the reference's step) on a bounded
    sample: the same workload (physics, velocity grid, dt) on a smaller
    spatial block, sized to ~budget_s seconds.  Returns (node-upd/s,
    description, threads)."""
    from oracle import oracle as O
    O.build()
    nthreads = threads or len(os.sched_getaffinity(0))
    O.set_num_threads(nthreads)
    import paper_2509_21832_b200 as mm
    side = 32
    while True:
        mesh = mm.PhaseMesh(space=(mm.Axis(0.0, side / cfg["nx"], side), mm.Axis(0.0, side / cfg["ny"], side)),
                            velocity=cfg["mesh"].velocity)
        prob = O.Problem2D(mesh, cfg["bc"], cfg["eps"], cfg["model"])
        Q = cfg["initial"](0, side, 0, side)
        G = np.zeros((side, side, 32, 32))
        O.step_2d_arrays(prob, Q, G, cfg["dt"])          # warm-up
        t0 = time.perf_counter()
        O.step_2d_arrays(prob, Q, G, cfg["dt"])
        dt1 = time.perf_counter() - t0
        if dt1 * 4 > budget_s or side >= min(cfg["nx"], cfg["ny"]):
            break
        side *= 2
    reps = max(1, int(budget_s / max(dt1, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(reps):
        Q2, G2, _ = O.step_2d_arrays(prob, Q, G, cfg["dt"])
    el = time.perf_counter() - t0
    nodes = side * side * 32 * 32 * reps
    desc = (f"oracle port of the reference step (C, OpenMP {nthreads} threads), "
            f"{side}x{side} block of the {cfg['name']} workload x 32^2 velocity, {reps} steps")
    return nodes / el, desc, nthreads, (prob, Q, G, side)


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    cfg = make_workload(args.config if args.config != "weak" else "c5")
    from oracle import oracle as O
    O.build()
    nthreads = len(os.sched_getaffinity(0))
    O.set_num_threads(nthreads)
    # size the per-step sample so warm-up + K steps fit in ~150 s
    rate, desc, th, (prob, Q, G, side) = cpu_sample(cfg, budget_s=2.0, threads=nthreads)
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    import paper_2509_21832_b200 as mm
    side_s = side
    while side_s > 8 and side_s * side_s * 1024 / rate > per_step_budget:
        side_s //= 2
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, side_s / cfg["nx"], side_s),
                               mm.Axis(0.0, side_s / cfg["ny"], side_s)),
                        velocity=cfg["mesh"].velocity)
    prob = O.Problem2D(mesh, cfg["bc"], cfg["eps"], cfg["model"])
    Qs = cfg["initial"](0, side_s, 0, side_s)
    Gs = np.zeros((side_s, side_s, 32, 32))
    for _ in range(args.warmup):
        Qs, Gs, _ = O.step_2d_arrays(prob, Qs, Gs, cfg["dt"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Qs, Gs, _ = O.step_2d_arrays(prob, Qs, Gs, cfg["dt"])
    el = time.perf_counter() - t0
    nodes = side_s * side_s * 1024 * args.steps
    value = nodes / el
    sample = (f"{side_s}x{side_s} block of the {cfg['name']} workload (same physics, 32^2 "
              f"velocity grid, dt) per step; oracle port of the reference kernels, C + OpenMP")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "sample": f"{side_s}x{side_s} cells x 32^2"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

RANK_GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}


# configs whose per-GPU block is fixed as N grows (the others split one domain)
WEAK_CONFIGS = ("c2", "weak", "c5w")


def rank_grid(world):
    if world in RANK_GRIDS:
        return RANK_GRIDS[world]
    px = int(math.sqrt(world))
    while world % px:
        px -= 1
    return (world // px, px)


def run_ours_multi(args, rank, world, local_rank):
    """Weak scaling over `world` GPUs (one process each): the N=1 workload's
    block per GPU, tiled into a px x py block grid of one periodic domain,
    with the two NCCL halo exchanges per step (G+Q ring, heat ring)."""
    import torch
    import torch.distributed as dist
    from paper_2509_21832_b200 import _native
    from paper_2509_21832_b200.parallel import (BlockStepper, DistExchange, make_plans,
                                                step_blocks)
    gloo = args.backend == "gloo"
    if gloo:
        # functional check of the multi-rank path on fewer GPUs than ranks:
        # exchanges go through pinned host memory, no kernel waits on another rank
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    px, py = rank_grid(world)
    cfg_name = args.config or "c2"
    cfg = make_workload(cfg_name, px=px, py=py)
    nx, ny, V = cfg["nx"], cfg["ny"], cfg["V"]
    plan = make_plans(nx, ny, (px, py), cfg["bc"])[rank]
    blk = BlockStepper(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"], (px, py), plan,
                       torch.device("cuda", local_rank))
    exch = DistExchange(plan, blk.bufs, staged=gloo)
    lib = _native.load()
    bx, by = plan.shape
    Q = torch.from_numpy(cfg["initial"](plan.i0, plan.i1, plan.j0, plan.j1)).cuda()
    G = torch.zeros((bx, by, 32, 32), dtype=torch.float64, device="cuda")
    st = [Q, G, torch.empty_like(Q), torch.empty_like(G),
          torch.empty((4, bx, by), dtype=torch.float64, device="cuda")]
    dt = cfg["dt"]
    dist.barrier()

    def steps(n):
        for _ in range(n):
            step_blocks([blk], exch, [st], dt)
            st[0], st[2] = st[2], st[0]
            st[1], st[3] = st[3], st[1]

    steps(args.warmup)
    torch.cuda.synchronize()
    blk.solver.check()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    lib.mm2d_reset_launch_count()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw0 = time.time()
    e0.record(stream)
    steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    tw1 = time.time()
    launches = int(lib.mm2d_launch_count())
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device="cpu" if gloo else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    dist.barrier()
    time.sleep(0.2)
    clocks.stop()
    blk.solver.check()
    clk = clocks.summary(tw0 - 0.05, tw1 + 0.05)
    value = nx * ny * V * args.steps / (ms / 1e3)
    ms_step = ms / args.steps
    peak, peak_src = measured_peak()
    step_bytes = bytes_per_step(nx, ny, V)
    step_gbs = step_bytes / (ms_step / 1e3) / 1e9
    # end to end: every rank uploads its block from pinned host memory,
    # runs one decomposed step and downloads the result
    Qh = st[0].cpu().pin_memory()
    Gh = st[1].cpu().pin_memory()
    Qo, Go = torch.empty_like(Qh).pin_memory(), torch.empty_like(Gh).pin_memory()
    Ho = torch.empty((4, bx, by), dtype=torch.float64).pin_memory()
    n_e2e = max(3, min(args.steps, 10))
    dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(n_e2e):
        st[0].copy_(Qh, non_blocking=True)
        st[1].copy_(Gh, non_blocking=True)
        step_blocks([blk], exch, [st], dt)
        Qo.copy_(st[2], non_blocking=True)
        Go.copy_(st[3], non_blocking=True)
        Ho.copy_(st[4], non_blocking=True)
    f1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([f0.elapsed_time(f1) / n_e2e], device="cpu" if gloo else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if cfg_name in WEAK_CONFIGS else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config initial conditions, g=0)",
        "config": {"workload": cfg["workload"], "nx": nx, "ny": ny, "nv1": 32, "nv2": 32,
                   "dt": dt, "parallelism": f"dd{px}x{py}",
                   "exchange": ("gloo via pinned host (functional test only)" if gloo else
                                "NCCL send/recv (torch.distributed)") +
                               ", Q ring, then the G ring overlapped with the interior "
                                 "micro CTAs, then the heat ring, per step",
                   "l2": "inputs larger than L2 (G per GPU = %.0f MiB)" % (bx * by * V * 8 / 2**20)},
        "roofline": {"bound": "hbm", "kernel": "full decomposed step",
                     "achieved": step_gbs / world, "peak": peak, "unit": "GB/s",
                     "frac": step_gbs / world / peak, "traffic": None, "peak_source": peak_src,
                     "note": "per-GPU algorithmic bytes of the whole step / step time"},
        "e2e": {"value": nx * ny * V / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": 8 * bx * by * (6 + V) * world,
                "d2h_bytes_per_step": 8 * bx * by * (6 + V + 4) * world, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_ours(args, rank, world, local_rank):
    if world > 1:
        return run_ours_multi(args, rank, world, local_rank)
    import torch
    import paper_2509_21832_b200 as mm
    from paper_2509_21832_b200 import _native
    from paper_2509_21832_b200.solver import Solver2D, _ptr

    torch.cuda.set_device(local_rank)
    dist = None
    cfg_name = args.config or "c2"
    cfg = make_workload(cfg_name)
    lib = _native.load()
    solver = Solver2D(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"])
    nx, ny, V = cfg["nx"], cfg["ny"], cfg["V"]
    S = solver.bx * solver.by
    Q0 = cfg["initial"](0, nx, 0, ny)
    Qa = torch.from_numpy(Q0).cuda()
    Ga = torch.zeros((nx, ny, 32, 32), dtype=torch.float64, device="cuda")
    Qb, Gb = solver.empty_state()
    H = torch.empty((4, nx, ny), dtype=torch.float64, device="cuda")
    dt = cfg["dt"]
    stream = torch.cuda.current_stream()

    # warm-up (also captures the CUDA graphs)
    solver.run(Qa, Ga, dt, max(args.warmup, 1), H_out=H, Q_b=Qb, G_b=Gb)
    torch.cuda.synchronize()
    solver.check()

    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    lib.mm2d_reset_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw0 = time.time()
    e0.record(stream)
    rc = lib.mm2d_run(solver.ctx, C.c_double(dt), int(args.steps))
    e1.record(stream)
    torch.cuda.synchronize()
    tw1 = time.time()
    if rc != 0:
        raise RuntimeError(_native.last_error(solver.ctx))
    launches = int(lib.mm2d_launch_count())
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    time.sleep(0.2)
    clocks.stop()
    solver.check()
    clk = clocks.summary(tw0 - 0.05, tw1 + 0.05)

    nodes = nx * ny * V * args.steps
    value = nodes / (ms / 1e3)
    ms_step = ms / args.steps

    # per-kernel device time (events on the launching stream), for the roofline
    kms = (C.c_double * 7)()
    lib.mm2d_set_stream(solver.ctx, C.c_void_p(stream.cuda_stream))
    rc = lib.mm2d_time_kernels(solver.ctx, C.c_double(dt), 5, kms)
    if rc != 0:
        raise RuntimeError(_native.last_error(solver.ctx))
    kms = list(kms)
    peak, peak_src = measured_peak()
    micro_bytes = 16.0 * S * V                      # G^n read + G^{n+1} write
    achieved = micro_bytes / (kms[2] / 1e3) / 1e9
    step_bytes = bytes_per_step(solver.bx, solver.by, V)
    step_gbs = step_bytes / (ms_step / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "micro_traffic.json"
    if tf.exists():
        try:
            td = json.loads(tf.read_text())
            if td.get("config") == cfg_name:
                traffic = td.get("bytes_per_launch")
        except Exception:
            traffic = None

    # end-to-end through the public API with host buffers: every step
    # uploads its state from pinned host memory, steps it (Solver2D.step ->
    # C ABI mm2d_step) and downloads the new state and heat tensor.  Steps
    # are pipelined over two device buffer sets and three streams so the
    # upload of step n+1 overlaps the download of step n (separate copy
    # engines); every byte still crosses PCIe inside the timed region.
    Qh = torch.from_numpy(Q0).pin_memory()
    Gh = torch.zeros((nx, ny, 32, 32), dtype=torch.float64).pin_memory()
    # two buffer sets (4 device copies of the state) when they fit in HBM,
    # else one (C5 at 2048^2: G alone is 32 GiB), which serialises the
    # upload of step n+1 behind the download of step n
    free_b = torch.cuda.mem_get_info()[0]
    n_sets = 2 if 4 * 8 * S * (V + 10) < 0.9 * free_b else 1
    outs_h = [(torch.empty_like(Qh).pin_memory(), torch.empty_like(Gh).pin_memory(),
               torch.empty((4, nx, ny), dtype=torch.float64).pin_memory()) for _ in range(n_sets)]
    ins_d = [solver.empty_state() for _ in range(n_sets)]
    outs_d = [solver.empty_state() + (torch.empty((4, nx, ny), dtype=torch.float64,
                                                  device="cuda"),) for _ in range(n_sets)]
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    n_e2e = max(4, min(args.steps, 20))

    def e2e_steps(n):
        for k in range(n):
            b = k % n_sets
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_free[b])
                ins_d[b][0].copy_(Qh, non_blocking=True)
                ins_d[b][1].copy_(Gh, non_blocking=True)
                ev_in[b].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[b])
                solver.step(ins_d[b][0], ins_d[b][1], dt, Q_out=outs_d[b][0],
                            G_out=outs_d[b][1], H_out=outs_d[b][2])
                ev_cmp[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[b])
                for hst, dev in zip(outs_h[b], outs_d[b]):
                    hst.copy_(dev, non_blocking=True)
                ev_free[b].record(s_out)

    for ev in ev_free[:n_sets]:
        ev.record(stream)
    e2e_steps(2)                                   # warm-up
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for st_ in (s_in, s_cmp, s_out):
        st_.wait_stream(stream)
    e2e_steps(n_e2e)
    for st_ in (s_in, s_cmp, s_out):
        stream.wait_stream(st_)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / n_e2e
    solver.check()
    e2e_value = nx * ny * V / (e2e_ms / 1e3)
    h2d = 8 * S * (6 + V)
    d2h = 8 * S * (6 + V + 4)
    del ins_d, outs_d
    torch.cuda.empty_cache()

    # end-to-end of a whole run the way a run_2d caller sees it: the host
    # state uploaded once, the config's step count advanced on the device
    # (Solver2D.run, one CUDA-graph replay), the final (Q, G) downloaded
    run_steps = cfg["run_steps"]
    Qr, Gr = Qa, Ga                                # the device-timed state is no longer needed

    def e2e_run():
        Qr.copy_(Qh, non_blocking=True)
        Gr.copy_(Gh, non_blocking=True)
        Qf, Gf = solver.run(Qr, Gr, dt, run_steps, H_out=H, Q_b=Qb, G_b=Gb)
        outs_h[0][0].copy_(Qf, non_blocking=True)
        outs_h[0][1].copy_(Gf, non_blocking=True)

    e2e_run()
    torch.cuda.synchronize()
    f0.record(stream)
    e2e_run()
    f1.record(stream)
    torch.cuda.synchronize()
    run_ms = f0.elapsed_time(f1)
    solver.check()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config initial conditions, g=0)",
        "config": {"workload": cfg["workload"], "nx": nx, "ny": ny, "nv1": 32, "nv2": 32,
                   "dt": dt, "parallelism": f"dd{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (G = %.0f MiB > 126 MB)" % (S * V * 8 / 2**20)},
        "roofline": {"bound": "hbm", "kernel": "k_micro (fused micro step)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": micro_bytes,
                     "launch_ms": kms[2], "peak_source": peak_src,
                     "step_achieved": step_gbs, "step_frac": step_gbs / peak,
                     # event intervals 0, 3 and 6 bracket no kernel any more (the ring
                     # fills are fused into k_prep / the sweeps, the SoA heat into
                     # k_macro_y)
                     "kernel_ms": {k: v for k, v in zip(
                         ["", "prep", "micro", "", "macro_x", "macro_y", ""], kms) if k}},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "path": "Solver2D.step (C ABI mm2d_step), pinned host state in/out every step, "
                        f"uploads/downloads pipelined over {n_sets} buffer set(s)"},
        "e2e_run": {"value": nx * ny * V * run_steps / (run_ms / 1e3), "unit": UNIT,
                    "steps": run_steps, "ms": run_ms, "h2d_bytes": h2d, "d2h_bytes": 8 * S * (6 + V),
                    "path": "one run_2d-style call: pinned host (Q, G) uploaded, Solver2D.run "
                            "(C ABI mm2d_run) for the config's step count, final (Q, G) downloaded"},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, desc, th, _ = cpu_sample(cfg, budget_s=12.0)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": th, "kind": "port",
                                "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional test of the multi-rank path on fewer GPUs than ranks")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        args.config = args.config or "c2"
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

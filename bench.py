#!/usr/bin/env python
"""Benchmark of the micro-macro ES-BGK 2D2V timestep on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c4s|c5|weak]
                  [--impl ours|reference]

A "step" is one full timestep of the hot path (prep -> fused micro kernel ->
macro KFVS/TR-BDF2) over the whole grid.  Default workload, at every N, is
BASELINE.json configs[4] (C5: 2048^2 x 32^2 periodic random Fourier, fp64,
eps = 1e-2): the largest configuration that fits one GPU, split into a
px x py block grid at N > 1 (strong scaling, the north star's 8-GPU target).
Metric: phase-space node-updates/s = nx*ny*nv1*nv2*K / seconds (device
time, CUDA events, max over ranks).  G is 32 GiB at C5 (> 126 MB L2), so
no L2 flush is needed between steps.

--impl reference times the REFERENCE's own CPU path -- the unmodified
micromacro package installed into baseline/_ref (compiled Cython backend)
-- on bounded samples of the same workload: run_parallel_2d over all usable
cores (the line's value) and the serial step_2d on one core; under
torchrun only rank 0 runs it.
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
    """Random smooth macro state of C5, a pure function of
    (seed, x, y) so every rank can build its own shard: three independent
    draws of 4 Fourier modes with integer (kx, ky), 1 <= |k| <= 4, phases
    U[0, 2 pi); psi = sum of the 4 cosines (|psi| <= 4).  rho = 1 + 0.1 psi0,
    u1 = 0.2 psi1, u2 = 0.2 psi2, T = 1 + 0.05 psi0, so rho >= 0.6, T >= 0.8."""
    rng = np.random.default_rng(seed)
    ks = []
    while len(ks) < 12:
        k = rng.integers(-4, 5, size=2)
        if 1 <= math.hypot(*k) <= 4:
            ks.append(k)
    ph = rng.uniform(0, 2 * np.pi, 12)

    def psi(m):
        return sum(np.cos(2 * np.pi * (ks[4 * m + q][0] * X + ks[4 * m + q][1] * Y) + ph[4 * m + q])
                   for q in range(4))

    p0, p1, p2 = psi(0), psi(1), psi(2)
    return 1.0 + 0.1 * p0, 0.2 * p1, 0.2 * p2, 1.0 + 0.05 * p0


DEFAULT_CONFIG = "c5"   # N=1: the largest single-GPU config (BASELINE configs[4], 2048^2)


def workload_spec(name, px=1, py=1, n=None, eps=None, seed=0):
    """Plain description of a BASELINE workload (no solver objects), shared
    by both arms, the golden generator and the parity tests.  ``n``
    overrides the cell count per axis (same generator, domain [0,1]^2);
    ``eps`` overrides the Knudsen number (C3 is run for three)."""
    Lx = Ly = 1.0
    if name == "c2":
        nx = ny = n or 256
        v, faces, ep, ic = (-7.0, 7.0), "periodic", 0.1, "wave"
        wl = f"C2 smooth periodic density wave {nx}^2 x 32^2 (BASELINE configs[1])"
        if px * py > 1 and n is None:
            wl = (f"C2 weak scaling: 256^2 x 32^2 per GPU, periodic wave tiled on "
                  f"{px}x{py} GPUs ({256 * px}x{256 * py} cells)")
            nx, ny = 256 * px, 256 * py
            Lx, Ly = float(px), float(py)
    elif name == "c3":
        nx = ny = n or 512
        v, faces, ep, ic = (-8.0, 8.0), "extrapolate", 1e-2, "riemann"
        wl = f"C3 four-quadrant Riemann {nx}^2 x 32^2 outflow(extrapolate)"
    elif name in ("c4", "c4s"):
        nx = ny = n or 1024
        v, ep, ic = (-8.0, 8.0), 5e-2, "bump"
        faces = "walls" if name == "c4" else "specular"
        wl = (f"C4 closed box, {'diffuse' if name == 'c4' else 'specular'} walls, "
              f"{nx}^2 x 32^2")
    elif name == "c5":
        nx = ny = n or 2048
        v, faces, ep, ic = (-7.0, 7.0), "periodic", 1e-2, "fourier"
        wl = f"C5 2048^2 x 32^2 periodic random Fourier (BASELINE configs[4], strong scaling)"
        if n:
            wl = f"C5 generator at {nx}^2 x 32^2"
    elif name in ("weak", "c5w"):
        nx, ny = (n or 1024) * px, (n or 1024) * py
        v, faces, ep, ic = (-7.0, 7.0), "periodic", 1e-2, "fourier"
        wl = f"C5 weak scaling {nx // px}^2 x 32^2 per GPU ({nx}x{ny} total)"
        Lx, Ly = float(px), float(py)
    else:
        raise SystemExit(f"unknown config {name}")
    if eps is not None:
        ep = float(eps)
    if name == "c3" or eps is not None:
        wl += f", eps={ep:g}"
    vmax = max(abs(v[0]), abs(v[1]))
    dt = 0.4 * min(Lx / nx, Ly / ny) / vmax
    # the run length each config names (C3: t = 0.1 at this dt)
    run_steps = {"c2": 100, "c3": int(np.ceil(0.1 / dt - 1e-9)), "c4": 200, "c4s": 200}.get(name, 50)
    return dict(name=name, workload=wl, nx=nx, ny=ny, Lx=Lx, Ly=Ly, vel=(v[0], v[1], 32),
                faces=faces, eps=ep, kind="esbgk_2d", nu=-0.5, ic=ic, seed=int(seed), dt=dt,
                V=32 * 32, run_steps=run_steps)


def initial_prims(spec, i0, i1, j0, j1):
    """(rho, u1, u2, T) of the config's initial condition on cells
    [i0, i1) x [j0, j1) (T_ab = T I, g = 0)."""
    nx, ny, Lx, Ly = spec["nx"], spec["ny"], spec["Lx"], spec["Ly"]
    x = (np.arange(i0, i1) + 0.5) * (Lx / nx)
    y = (np.arange(j0, j1) + 0.5) * (Ly / ny)
    X, Y = np.meshgrid(x, y, indexing="ij")
    one = np.ones_like(X)
    ic = spec["ic"]
    if ic == "wave":
        rho = 1.0 + 0.2 * np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)
        return rho, 0.5 * one, 0.5 * one, one
    if ic == "riemann":
        north, east = Y >= 0.5, X >= 0.5
        rho = np.where(north, np.where(east, 1.0, 0.5), np.where(east, 0.5, 0.25))
        u1 = np.where(north, np.where(east, 0.0, 0.5), np.where(east, 0.0, 0.5))
        u2 = np.where(north, 0.0, 0.5)
        T = np.where(north, np.where(east, 1.0, 0.8), np.where(east, 0.8, 0.6))
        return rho, u1, u2, T
    if ic == "bump":
        rho = 1.0 + 0.5 * np.exp(-((X - 0.3) ** 2 + (Y - 0.6) ** 2) / 0.01)
        return rho, 0 * one, 0 * one, one
    return c5_fields(spec["seed"], X, Y)


def public_config(spec, world=1, px=1, py=1):
    """The `config` object of the JSON line: identical in both arms."""
    S = spec["nx"] * spec["ny"] // max(1, px * py)
    return {"workload": spec["workload"], "nx": spec["nx"], "ny": spec["ny"], "nv1": 32,
            "nv2": 32, "eps": spec["eps"], "nu": spec["nu"], "dt": spec["dt"],
            "seed": spec["seed"] if spec["ic"] == "fourier" else None,
            "parallelism": f"dd{px}x{py}" if world > 1 else "single",
            "l2": "inputs larger than L2 (G per GPU = %.0f MiB > 126 MB), no flush needed"
                  % (S * spec["V"] * 8 / 2**20)}


def make_workload(name, n_gpus=1, px=1, py=1, n=None, eps=None, seed=0):
    """The workload as this framework's solver objects."""
    import paper_2509_21832_b200 as mm
    spec = workload_spec(name, px, py, n=n, eps=eps, seed=seed)
    lo, hi, nv = spec["vel"]
    mesh = mm.PhaseMesh(space=(mm.Axis(0.0, spec["Lx"], spec["nx"]),
                               mm.Axis(0.0, spec["Ly"], spec["ny"])),
                        velocity=(mm.Axis(lo, hi, nv), mm.Axis(lo, hi, nv)))
    faces = spec["faces"]
    if faces == "periodic":
        bc = mm.BoundarySpec2D(mm.PERIODIC, mm.PERIODIC, mm.PERIODIC, mm.PERIODIC)
    elif faces == "extrapolate":
        bc = mm.BoundarySpec2D(mm.EXTRAPOLATE, mm.EXTRAPOLATE, mm.EXTRAPOLATE, mm.EXTRAPOLATE)
    elif faces == "specular":
        bc = mm.BoundarySpec2D(mm.SPECULAR, mm.SPECULAR, mm.SPECULAR, mm.SPECULAR)
    else:
        w = mm.WallSpec(1.0, 0.0)
        bc = mm.BoundarySpec2D(w, w, w, w)
    model = mm.CollisionModel(spec["kind"], nu=spec["nu"])

    def initial(i0, i1, j0, j1):
        rho, u1, u2, T = initial_prims(spec, i0, i1, j0, j1)
        return mm.conserved_2d(rho, u1, u2, T, 0 * T, T)

    return dict(spec, mesh=mesh, bc=bc, model=model, initial=initial)


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
# CPU arm: the reference's own CPU path (baseline/_ref), the oracle port beside it
# ---------------------------------------------------------------------------

REF_DIR = ROOT / "baseline" / "_ref"


def cpu_info():
    logical = os.cpu_count() or 1
    usable = len(os.sched_getaffinity(0))
    try:
        import psutil
        physical = psutil.cpu_count(logical=False)
    except Exception:  # pragma: no cover
        physical = None
    return {"logical": logical, "usable": usable, "physical": physical}


def import_reference():
    """The unmodified reference package, installed into baseline/_ref by
    oracle/build_ref.sh (pip install of /root/reference/pkg, compiled Cython
    backend).  Returns (namespace, None) or (None, why)."""
    if not (REF_DIR / "micromacro").is_dir():
        return None, "baseline/_ref is missing (oracle/build_ref.sh installs it)"
    os.environ["MICROMACRO_BACKEND"] = "compiled"
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import importlib
        K = importlib.import_module("micromacro._kernels")
        if K.backend_name != "compiled":
            return None, f"reference backend is {K.backend_name!r}, not 'compiled'"
        from types import SimpleNamespace
        ns = SimpleNamespace(
            mesh=importlib.import_module("micromacro.mesh"),
            boundary=importlib.import_module("micromacro.boundary"),
            gas=importlib.import_module("micromacro.gas_state"),
            loop=importlib.import_module("micromacro.runner.loop"),
            parallel=importlib.import_module("micromacro.runner.parallel"),
            backend=K.backend_name)
        return ns, None
    except Exception as exc:  # noqa: BLE001
        return None, f"reference import failed: {exc!r}"


def reference_problem(R, spec, side_x, side_y):
    """The reference's own objects for a side_x x side_y block of the
    workload: the same dx, dt, velocity grid, faces and physics."""
    if spec["faces"] == "specular":
        raise SystemExit("specular walls are an extension; the reference has no CPU path for them")
    dx, dy = spec["Lx"] / spec["nx"], spec["Ly"] / spec["ny"]
    lo, hi, nv = spec["vel"]
    mesh = R.mesh.PhaseMesh(space=(R.mesh.Axis(0.0, side_x * dx, side_x),
                                   R.mesh.Axis(0.0, side_y * dy, side_y)),
                            velocity=(R.mesh.Axis(lo, hi, nv), R.mesh.Axis(lo, hi, nv)))
    B = R.boundary
    if spec["faces"] == "periodic":
        bc = B.BoundarySpec2D(B.PERIODIC, B.PERIODIC, B.PERIODIC, B.PERIODIC)
    elif spec["faces"] == "extrapolate":
        bc = B.BoundarySpec2D(B.EXTRAPOLATE, B.EXTRAPOLATE, B.EXTRAPOLATE, B.EXTRAPOLATE)
    else:
        w = B.WallSpec(temperature=1.0, velocity=0.0)
        bc = B.BoundarySpec2D(w, w, w, w)
    model = R.gas.CollisionModel(spec["kind"], nu=spec["nu"])
    rho, u1, u2, T = initial_prims(spec, 0, side_x, 0, side_y)
    Q = R.gas.conserved_2d(rho, u1, u2, T, 0 * T, T)
    G = np.zeros((side_x, side_y, nv, nv))
    return mesh, bc, model, Q, G


def worker_grid(n):
    """rows x cols = n with rows <= cols, as square as possible."""
    r = int(math.sqrt(n))
    while n % r:
        r -= 1
    return r, n // r


def time_reference(spec, steps, warmup, serial_steps=3, log=None):
    """Time the reference's CPU path on bounded samples of the workload.

    (i) all usable cores: run_parallel_2d (parallel.py:404-473) with a
        rows x cols worker grid, one worker per core, on a block of about
        256^2 cells; its `seconds` include fork/join, so it runs `warmup`
        and `warmup + steps` steps and the per-step time is the difference;
    (ii) one core: the serial step_2d (loop.py:82-111) on a 128^2 block, one
        warm-up step then `serial_steps` timed steps.
    Returns a dict (value = (i) in node-updates/s)."""
    R, why = import_reference()
    if R is None:
        return None, why
    info = cpu_info()
    V = spec["V"]
    out = {"cpu": info, "backend": R.backend}
    # (i) all cores
    rows, cols = worker_grid(info["usable"])
    bx = max(16, -(-256 // rows))
    by = max(16, -(-256 // cols))
    sx, sy = rows * bx, cols * by
    need = 8 * sx * sy * (2 * V + 16) * 1.1
    try:
        import shutil
        shm_free = shutil.disk_usage("/dev/shm").free
    except Exception:  # pragma: no cover
        shm_free = 0
    while need > shm_free and sx > rows * 16:
        bx, by = max(16, bx // 2), max(16, by // 2)
        sx, sy = rows * bx, cols * by
        need = 8 * sx * sy * (2 * V + 16) * 1.1
    if need <= shm_free:
        mesh, bc, model, Q, G = reference_problem(R, spec, sx, sy)
        run = R.parallel.run_parallel_2d
        n1, n2 = max(1, warmup), max(1, warmup) + steps
        _, _, _, t1 = run(mesh, bc, spec["eps"], model, Q, G, spec["dt"], n1, grid=(rows, cols))
        _, _, _, t2 = run(mesh, bc, spec["eps"], model, Q, G, spec["dt"], n2, grid=(rows, cols))
        per = max(t2 - t1, 1e-9) / (n2 - n1)
        out["all_cores"] = {
            "value": sx * sy * V / per, "unit": UNIT, "cores": rows * cols,
            "sample": (f"reference run_parallel_2d (compiled backend), {rows}x{cols} worker grid "
                       f"(one process per usable core) on a {sx}x{sy} block of the "
                       f"{spec['name']} workload (same dx, dt, 32^2 velocity grid, eps, nu), "
                       f"per-step time = (t({n2}) - t({n1})) / {n2 - n1} to remove fork/join"),
            "ms_per_step": 1e3 * per}
    else:
        out["all_cores"] = None
        out["all_cores_skipped"] = f"/dev/shm has {shm_free} bytes free, needs {int(need)}"
    # (ii) one core
    mesh, bc, model, Q, G = reference_problem(R, spec, 128, 128)
    st = R.loop.State2D(t=0.0, Q=Q, G=G)
    st = R.loop.step_2d(st, mesh, bc, spec["eps"], model, spec["dt"])
    t0 = time.perf_counter()
    for _ in range(serial_steps):
        st = R.loop.step_2d(st, mesh, bc, spec["eps"], model, spec["dt"])
    per1 = (time.perf_counter() - t0) / serial_steps
    out["one_core"] = {"value": 128 * 128 * V / per1, "unit": UNIT, "cores": 1,
                       "sample": (f"reference serial step_2d (compiled backend), 128x128 block of "
                                  f"the {spec['name']} workload, 1 warm-up + {serial_steps} "
                                  f"timed steps"), "ms_per_step": 1e3 * per1}
    return out, None


def time_port(spec, budget_s=3.0):
    """The oracle port (C + OpenMP restatement of the reference step, test
    infrastructure) on a bounded block of the workload: a secondary line."""
    from oracle import oracle as O
    import paper_2509_21832_b200 as mm   # host-side problem objects only
    O.build()
    nthreads = len(os.sched_getaffinity(0))
    O.set_num_threads(nthreads)
    cfg = make_workload(spec["name"], n=None if spec["name"] != "c3" else spec["nx"],
                        eps=spec["eps"], seed=spec["seed"])
    side = 64
    while True:
        mesh = mm.PhaseMesh(space=(mm.Axis(0.0, side / spec["nx"], side),
                                   mm.Axis(0.0, side / spec["ny"], side)),
                            velocity=cfg["mesh"].velocity)
        prob = O.Problem2D(mesh, cfg["bc"], spec["eps"], cfg["model"])
        Q = cfg["initial"](0, side, 0, side)
        G = np.zeros((side, side, 32, 32))
        O.step_2d_arrays(prob, Q, G, spec["dt"])
        t0 = time.perf_counter()
        O.step_2d_arrays(prob, Q, G, spec["dt"])
        dt1 = time.perf_counter() - t0
        if dt1 * 4 > budget_s or side >= 256:
            break
        side *= 2
    reps = max(1, int(budget_s / max(dt1, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(reps):
        O.step_2d_arrays(prob, Q, G, spec["dt"])
    el = time.perf_counter() - t0
    return {"value": side * side * 1024 * reps / el, "unit": UNIT, "cores": nthreads,
            "kind": "port",
            "sample": (f"oracle port of the reference step (C, OpenMP {nthreads} threads), "
                       f"{side}x{side} block, {reps} steps")}


def cpu_baseline_of(res):
    """The `cpu_baseline` object from a time_reference() result."""
    head = res["all_cores"] or res["one_core"]
    return {"value": head["value"], "unit": UNIT, "cores": head["cores"], "kind": "reference",
            "sample": head["sample"], "cpu": res["cpu"],
            "one_core": {k: res["one_core"][k] for k in ("value", "sample", "ms_per_step")},
            **({"port": res["port"]} if res.get("port") else {})}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    name = args.config or DEFAULT_CONFIG
    px, py = rank_grid(world) if world > 1 else (1, 1)
    spec = workload_spec(name, px, py, eps=args.eps, seed=args.seed)
    res, why = time_reference(spec, args.steps, args.warmup,
                              serial_steps=args.serial_steps)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    if not args.no_port:
        try:
            res["port"] = time_port(spec)
        except Exception as exc:  # noqa: BLE001
            res["port"] = {"error": repr(exc)}
    cb = cpu_baseline_of(res)
    head = res["all_cores"] or res["one_core"]
    line = {
        "impl": "reference", "metric": METRIC, "value": head["value"], "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "weak" if name in WEAK_CONFIGS else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config initial conditions, g=0)",
        "config": public_config(spec, world, px, py),
        "cpu_baseline": cb,
        "e2e": {"value": head["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
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
    from paper_2509_21832_b200.parallel import (BlockStepper, DistExchange, IpcPeers, make_plans,
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
    cfg_name = args.config or DEFAULT_CONFIG
    cfg = make_workload(cfg_name, px=px, py=py, eps=args.eps, seed=args.seed)
    nx, ny, V = cfg["nx"], cfg["ny"], cfg["V"]
    plan = make_plans(nx, ny, (px, py), cfg["bc"])[rank]
    blk = BlockStepper(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"], (px, py), plan,
                       torch.device("cuda", local_rank))
    exch = DistExchange(plan, blk.bufs, staged=gloo)
    lib = _native.load()
    bx, by = plan.shape
    Q = torch.from_numpy(cfg["initial"](plan.i0, plan.i1, plan.j0, plan.j1)).cuda()
    # peer form of the G halo: every rank maps its neighbours' G buffers
    # (CUDA IPC) and its micro kernel reads the ghost cells in place over
    # NVLink; all ranks must agree, so one failed mapping selects the packed
    # NCCL ring everywhere
    peers = None
    if args.halo == "peer" and any(s is not None for s in plan.slots):
        peers = IpcPeers(blk.solver, plan, (bx, by, 32, 32))
        flag = torch.tensor([0 if peers.failed else 1], device="cpu" if gloo else "cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            if peers.failed and rank == 0:
                print(f"bench: peer-form halo unavailable ({peers.failed}); packed ring",
                      file=sys.stderr)
            peers.close()
            peers = None
    if peers is not None:
        G, Gb = peers.tensors
        G.zero_()
    else:
        G = torch.zeros((bx, by, 32, 32), dtype=torch.float64, device="cuda")
        Gb = torch.empty_like(G)
    st = [Q, G, torch.empty_like(Q), Gb,
          torch.empty((4, bx, by), dtype=torch.float64, device="cuda")]
    dt = cfg["dt"]
    par = [0]
    dist.barrier()

    def steps(n):
        for _ in range(n):
            step_blocks([blk], exch, [st], dt,
                        peers=[peers.views(par[0])] if peers is not None else None)
            st[0], st[2] = st[2], st[0]
            st[1], st[3] = st[3], st[1]
            par[0] ^= 1

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
        "config": public_config(cfg, world, px, py),
        "exchange": ("gloo via pinned host (functional test only)" if gloo else
                     "NCCL send/recv (torch.distributed)") +
                    (", Q ring, G ghost cells read in place from the neighbours' arrays "
                     "(CUDA-IPC peer memory), then the heat ring, per step" if peers is not None
                     else ", Q ring, then the G ring overlapped with the interior micro CTAs, "
                          "then the heat ring, per step"),
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
    if peers is not None:
        del st, G, Gb
        peers.close()
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
    cfg_name = args.config or DEFAULT_CONFIG
    cfg = make_workload(cfg_name, eps=args.eps, seed=args.seed)
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
    rc = lib.mm2d_time_kernels(solver.ctx, C.c_double(dt), max(3, min(args.steps, 200)), kms)
    if rc != 0:
        raise RuntimeError(_native.last_error(solver.ctx))
    kms = list(kms)
    peak, peak_src = measured_peak()
    micro_bytes = 16.0 * S * V                      # G^n read + G^{n+1} write
    achieved = micro_bytes / (kms[2] / 1e3) / 1e9
    step_bytes = bytes_per_step(solver.bx, solver.by, V)
    step_gbs = step_bytes / (ms_step / 1e3) / 1e9
    traffic, traffic_note = micro_traffic(lib, cfg_name)
    if args.no_e2e:   # A/B timing runs: device numbers only
        print(json.dumps({"metric": METRIC, "value": value, "ms_per_step": ms_step,
                          "config": public_config(cfg, world), "clocks": clk,
                          "roofline": {"frac": achieved / peak, "launch_ms": kms[2],
                                       "step_frac": step_gbs / peak,
                                       "kernel_ms": {k: v for k, v in zip(
                                           ["", "prep", "micro", "", "macro_x", "macro_y", ""],
                                           kms) if k}}}), flush=True)
        return

    # end to end of a whole run the way a run_2d caller sees it: the host
    # state uploaded once, the config's step count advanced on the device
    # (Solver2D.run, one CUDA-graph replay), the final (Q, G) downloaded
    Qh = torch.from_numpy(Q0).pin_memory()
    Gh = torch.zeros((nx, ny, 32, 32), dtype=torch.float64).pin_memory()
    Qo_h = torch.empty_like(Qh).pin_memory()
    Go_h = torch.empty_like(Gh).pin_memory()
    Ho_h = torch.empty((4, nx, ny), dtype=torch.float64).pin_memory()
    run_steps = cfg["run_steps"]
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def e2e_run():
        Qa.copy_(Qh, non_blocking=True)
        Ga.copy_(Gh, non_blocking=True)
        Qf, Gf = solver.run(Qa, Ga, dt, run_steps, H_out=H, Q_b=Qb, G_b=Gb)
        Qo_h.copy_(Qf, non_blocking=True)
        Go_h.copy_(Gf, non_blocking=True)

    e2e_run()
    torch.cuda.synchronize()
    f0.record(stream)
    e2e_run()
    f1.record(stream)
    torch.cuda.synchronize()
    run_ms = f0.elapsed_time(f1)
    solver.check()
    # the device-timed state is no longer needed: free it for the e2e sets
    del Qa, Ga, Qb, Gb
    solver.close()
    solver = Solver2D(cfg["mesh"], cfg["bc"], cfg["eps"], cfg["model"])
    torch.cuda.empty_cache()

    # end to end through the public API with host buffers: every step
    # uploads its state from pinned host memory, steps it (Solver2D.step ->
    # C ABI mm2d_step) and downloads the new state and heat tensor.  Steps
    # are pipelined over two device buffer sets and three streams so the
    # upload of step n+1 overlaps the download of step n (separate copy
    # engines); every byte still crosses PCIe inside the timed region.  One
    # pinned host input and one output set serve both device sets (the copies
    # on each stream are serialised anyway).
    free_b = torch.cuda.mem_get_info()[0]
    n_sets = 2 if 4 * 8 * S * (V + 10) < 0.92 * free_b else 1
    ins_d = [solver.empty_state() for _ in range(n_sets)]
    outs_d = [solver.empty_state() + (torch.empty((4, nx, ny), dtype=torch.float64,
                                                  device="cuda"),) for _ in range(n_sets)]
    outs_h = (Qo_h, Go_h, Ho_h)
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
                for hst, dev in zip(outs_h, outs_d[b]):
                    hst.copy_(dev, non_blocking=True)
                ev_free[b].record(s_out)

    for ev in ev_free[:n_sets]:
        ev.record(stream)
    e2e_steps(2)                                   # warm-up
    torch.cuda.synchronize()
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

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if cfg_name in WEAK_CONFIGS else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config initial conditions, g=0)",
        "config": public_config(cfg, world),
        "roofline": {"bound": "hbm", "kernel": "k_micro32 (fused micro step)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_note,
                     "algorithmic_bytes_per_launch": micro_bytes,
                     "launch_ms": kms[2], "peak_source": peak_src,
                     "kernel_version": int(lib.mm2d_kernel_version()),
                     "step_achieved": step_gbs, "step_frac": step_gbs / peak,
                     "kernel_ms_source": ("CUDA events recorded inside one captured graph of "
                                          f"{args.steps} steps (the timed path plus event nodes)"),
                     "kernel_ms": {k: v for k, v in zip(
                         ["", "prep", "micro", "", "macro_x", "macro_y", ""], kms) if k}},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "path": "Solver2D.step (C ABI mm2d_step), pinned host state in/out every step, "
                        f"uploads/downloads pipelined over {n_sets} device buffer set(s)"},
        "e2e_run": {"value": nx * ny * V * run_steps / (run_ms / 1e3), "unit": UNIT,
                    "steps": run_steps, "ms": run_ms, "h2d_bytes": h2d, "d2h_bytes": 8 * S * (6 + V),
                    "path": "one run_2d-style call: pinned host (Q, G) uploaded, Solver2D.run "
                            "(C ABI mm2d_run) for the config's step count, final (Q, G) downloaded"},
        "gpu_launches": launches,
        "clocks": clk,
    }
    solver.close()
    del Qh, Gh, Qo_h, Go_h, Ho_h, outs_h
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = reference_subprocess(cfg_name, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def micro_traffic(lib, cfg_name):
    """DRAM bytes per k_micro32 launch from the committed ncu capture, used
    only when it was taken on this kernel version and this config."""
    tf = ROOT / "profiles" / "micro_traffic.json"
    ver = int(lib.mm2d_kernel_version())
    if not tf.exists():
        return None, "no ncu capture committed"
    try:
        td = json.loads(tf.read_text())
    except Exception as exc:  # noqa: BLE001
        return None, f"unreadable profiles/micro_traffic.json: {exc!r}"
    for rec in td.get("captures", []):
        if rec.get("config") == cfg_name and int(rec.get("kernel_version", -1)) == ver:
            return rec["bytes_per_launch"], (f"ncu --set full, dram__bytes_read.sum + "
                                             f"dram__bytes_write.sum, kernel v{ver}, "
                                             f"{rec.get('report', '')}")
    return None, f"no ncu capture of kernel v{ver} on {cfg_name} in profiles/micro_traffic.json"


def reference_subprocess(cfg_name, args):
    """cpu_baseline of the N=1 line: the reference arm in a fresh process
    (no CUDA context), on a shorter bounded sample."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", cfg_name,
           "--steps", "4", "--warmup", "3", "--serial-steps", "2", "--no-port",
           "--seed", str(args.seed)]
    if args.eps is not None:
        cmd += ["--eps", str(args.eps)]
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
        for ln in r.stdout.splitlines()[::-1]:
            if ln.startswith("{"):
                d = json.loads(ln)
                if "cpu_baseline" in d:
                    return d["cpu_baseline"]
                return {"value": None, "unit": UNIT, "unavailable": d.get("unavailable")}
        return {"value": None, "unit": UNIT,
                "unavailable": f"reference arm printed no line (rc {r.returncode}): "
                               f"{r.stderr[-300:]}"}
    except subprocess.TimeoutExpired:
        return {"value": None, "unit": UNIT, "unavailable": "reference arm timed out"}


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
    ap.add_argument("--halo", default="peer", choices=["peer", "packed"],
                    help="multi-GPU G halo: peer = ghost cells read in place from the neighbours' "
                         "arrays over NVLink (CUDA IPC); packed = packed NCCL ring")
    ap.add_argument("--eps", type=float, default=None, help="override the config's Knudsen number")
    ap.add_argument("--seed", type=int, default=0, help="C5 initial-condition seed")
    ap.add_argument("--serial-steps", type=int, default=3,
                    help="reference arm: timed serial step_2d steps on one core")
    ap.add_argument("--no-port", action="store_true", help="reference arm: skip the port line")
    ap.add_argument("--no-e2e", action="store_true",
                    help="A/B timing: print the device-timed numbers only (no e2e, no CPU arm)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

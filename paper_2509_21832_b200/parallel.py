"""Block domain decomposition of the 2D step across GPUs.

Drop-in for the reference's worker-grid runner
(pkg/src/micromacro/runner/parallel.py): ``HaloPlan`` / ``make_plans``
(50-93) partition the (nx, ny) grid into a rows x cols block grid with the
same rank numbering and periodic neighbour wrap; ``run_parallel_2d``
(404-473) keeps its signature and return value.

Where the reference forks CPU workers that read one-cell rings straight out
of POSIX shared memory (extract_ring, 109-150) and meet at two barriers per
step (384-394), each block here is a libmm2d context on a GPU and the rings
are exchanged explicitly, twice per step, exactly at the reference's two
barrier points:

  1. before the micro phase: the G ring (V doubles per cell) and the Q ring
     (6 doubles per cell) from up to 8 neighbours (faces + corners);
  2. between the micro and the macro phase: the heat-tensor ring (4 doubles
     per cell).

Two transports implement the same slot protocol (slot s of a block goes to
its neighbour in direction s and lands in that neighbour's slot opposite(s)):

  * ``DistExchange``: one process per GPU, ``torch.distributed`` batched
    isend/irecv -- NCCL over NVLink/NVSwitch on B200, gloo on CPU (tests);
  * ``LoopbackExchange``: all blocks in one process, device-to-device copies
    between the contexts' staging buffers (peer copies when the blocks sit
    on different GPUs).

Per-cell arithmetic does not depend on the decomposition, so results are
bitwise identical to the single-block step (the property the reference's
test_parallel.py:96-110 pins for its worker grid).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from .boundary import PERIODIC
from .errors import ConfigurationError

# slot order shared with the C ABI (include/mm2d.h): faces then corners
SLOTS = ("left", "right", "bottom", "top", "bottom_left", "bottom_right", "top_left",
         "top_right")
SLOT_DIR = ((-1, 0), (1, 0), (0, -1), (0, 1), (-1, -1), (1, -1), (-1, 1), (1, 1))
OPPOSITE = (1, 0, 3, 2, 7, 6, 5, 4)
FIELD_G, FIELD_Q, FIELD_H = 0, 1, 2


@dataclass(frozen=True)
class HaloPlan:
    """One block's extent and its exchange neighbours (rank per slot, None
    for a physical face or a face wrapped locally)."""

    rank: int
    grid: tuple
    pos: tuple
    i0: int
    i1: int
    j0: int
    j1: int
    neighbors: dict          # face name -> rank or None (reference naming)
    slots: tuple             # 8 entries: neighbour rank per exchange slot

    @property
    def shape(self):
        return (self.i1 - self.i0, self.j1 - self.j0)


def make_plans(nx, ny, grid, bc):
    """Block plans in the reference's numbering: rank = r * cols + c for
    block (r, c), x split into `rows`, y into `cols` (parallel.py:69-93)."""
    rows, cols = grid
    if rows < 1 or cols < 1 or nx % rows != 0 or ny % cols != 0:
        raise ConfigurationError(
            f"worker grid {rows}x{cols} must divide the spatial grid {nx}x{ny}")
    bx, by = nx // rows, ny // cols
    xper = bc.left == PERIODIC
    yper = bc.bottom == PERIODIC

    def nb_face(r, c, dr, dc):
        rr, cc = r + dr, c + dc
        if 0 <= rr < rows and 0 <= cc < cols:
            return rr * cols + cc
        if dr and xper:
            return (rr % rows) * cols + cc
        if dc and yper:
            return rr * cols + (cc % cols)
        return None

    plans = []
    for r in range(rows):
        for c in range(cols):
            faces = {"left": nb_face(r, c, -1, 0), "right": nb_face(r, c, 1, 0),
                     "bottom": nb_face(r, c, 0, -1), "top": nb_face(r, c, 0, 1)}
            # exchange slots: a face is exchanged iff it is an interior face or
            # periodic across more than one block along that axis (a single
            # block wraps locally); corners iff both adjacent faces are
            xs = [faces["left"] if (r > 0 or (xper and rows > 1)) else None,
                  faces["right"] if (r < rows - 1 or (xper and rows > 1)) else None]
            ys = [faces["bottom"] if (c > 0 or (yper and cols > 1)) else None,
                  faces["top"] if (c < cols - 1 or (yper and cols > 1)) else None]
            slot = xs + ys
            for dr, dc in SLOT_DIR[4:]:
                ok = slot[0 if dr < 0 else 1] is not None and slot[2 if dc < 0 else 3] is not None
                slot.append(((r + dr) % rows) * cols + ((c + dc) % cols) if ok else None)
            plans.append(HaloPlan(rank=r * cols + c, grid=(rows, cols), pos=(r, c),
                                  i0=r * bx, i1=(r + 1) * bx, j0=c * by, j1=(c + 1) * by,
                                  neighbors=faces, slots=tuple(slot)))
    return plans


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class DistExchange:
    """Slot exchange over torch.distributed point-to-point (one block per
    rank).  ``bufs[field][slot] = (send, recv)`` tensors (None when the slot
    is inactive).  Sends are posted in slot order and receives in slot order
    of the opposite direction, so the matching between any pair of ranks is
    well defined even when one neighbour occupies several slots (periodic
    wrap over two blocks).

    With ``staged=True`` (a backend without device P2P, e.g. gloo driving
    device buffers in tests) every slot goes through pinned host mirrors."""

    def __init__(self, plan: HaloPlan, bufs, group=None, staged=False):
        self.plan = plan
        self.bufs = bufs
        self.group = group
        self.staged = staged
        self._host = {}

    def _mirror(self, t):
        key = t.data_ptr()
        if key not in self._host:
            import torch
            self._host[key] = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        return self._host[key]

    def exchange(self, field):
        self.finish(self.start(field))

    def start(self, field):
        """Post the field's sends and receives; returns the handle ``finish``
        completes.  Over NCCL the transfers run on the communicator's stream
        while the caller keeps enqueueing work (the interior micro CTAs)."""
        import torch.distributed as dist
        ops, back = [], []
        for s in range(8):
            peer = self.plan.slots[s]
            send, _ = self.bufs[field][s]
            if peer is not None and send is not None:
                if self.staged:
                    h = self._mirror(send)
                    h.copy_(send)
                    send = h
                ops.append(dist.P2POp(dist.isend, send, peer, self.group))
        for s in range(8):
            o = OPPOSITE[s]
            peer = self.plan.slots[o]
            _, recv = self.bufs[field][o]
            if peer is not None and recv is not None:
                if self.staged:
                    h = self._mirror(recv)
                    back.append((recv, h))
                    recv = h
                ops.append(dist.P2POp(dist.irecv, recv, peer, self.group))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        if self.staged:
            self.finish((reqs, back))
            return ([], [])
        return (reqs, back)

    def finish(self, handle):
        """Make the current stream wait for a started exchange (NCCL: a
        stream-side wait, the host does not block)."""
        reqs, back = handle
        for req in reqs:
            req.wait()
        for dev, h in back:
            dev.copy_(h)


class LoopbackExchange:
    """Slot exchange between blocks held by one process: copy every active
    send slot into the neighbour's opposite receive slot.

    Ordering is stream-side only (no host synchronisation): a copy runs on
    the destination device's current stream after an event recorded on the
    source device's current stream (so after the pack kernel that filled the
    send buffer), and the source stream waits for the copies out of its
    buffers before anything it enqueues next (the next pack)."""

    def __init__(self, plans, bufs_per_block):
        self.plans = plans
        self.bufs = bufs_per_block

    def exchange(self, field):
        import torch
        copies = []
        for p in self.plans:
            for s in range(8):
                peer = p.slots[s]
                if peer is None:
                    continue
                send, _ = self.bufs[p.rank][field][s]
                _, recv = self.bufs[peer][field][OPPOSITE[s]]
                if send is not None and recv is not None:
                    copies.append((send, recv))
        cross = [(a, b) for a, b in copies if a.device != b.device]
        if not cross:
            for send, recv in copies:
                recv.copy_(send, non_blocking=True)
            return
        devs = sorted({t.device.index for c in copies for t in c})
        ready = {}
        for d in devs:
            with torch.cuda.device(d):
                ready[d] = torch.cuda.Event()
                ready[d].record()
        waited = set()
        for send, recv in copies:
            a, b = send.device.index, recv.device.index
            with torch.cuda.device(b):
                if a != b and (a, b) not in waited:
                    torch.cuda.current_stream().wait_event(ready[a])
                    waited.add((a, b))
                recv.copy_(send, non_blocking=True)
        done = {}
        for d in devs:
            with torch.cuda.device(d):
                done[d] = torch.cuda.Event()
                done[d].record()
        for a, b in waited:
            with torch.cuda.device(a):
                torch.cuda.current_stream().wait_event(done[b])

    def start(self, field):
        self.exchange(field)

    def finish(self, handle):
        pass


# ---------------------------------------------------------------------------
# device blocks
# ---------------------------------------------------------------------------

class _CAI:
    """Minimal __cuda_array_interface__ view of a device pointer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def halo_buffers(solver):
    """(send, recv) tensors per (field, slot), viewing the context's staging
    buffers (None for inactive slots)."""
    import torch
    lib, ctx = solver.lib, solver.ctx
    out = []
    for f in range(3):
        row = []
        for s in range(8):
            sp, rp, n = C.c_void_p(), C.c_void_p(), C.c_longlong()
            rc = lib.mm2d_halo_info(ctx, f, s, C.byref(sp), C.byref(rp), C.byref(n))
            if rc != 0:
                raise RuntimeError(f"mm2d_halo_info failed: {rc}")
            if n.value == 0:
                row.append((None, None))
                continue
            with torch.cuda.device(solver.device):
                st = torch.as_tensor(_CAI(sp.value, n.value), device=solver.device)
                rt = torch.as_tensor(_CAI(rp.value, n.value), device=solver.device)
            row.append((st, rt))
        out.append(row)
    return out


class BlockStepper:
    """One block of a decomposition on one GPU: a libmm2d context plus the
    exchange protocol around its two step phases."""

    def __init__(self, mesh, bc, eps, model, grid, plan: HaloPlan, device):
        from .solver import Solver2D
        self.plan = plan
        self.solver = Solver2D(mesh, bc, eps, model, grid=grid, rank=plan.pos, device=device)
        self.bufs = halo_buffers(self.solver)
        import torch
        with torch.cuda.device(device):
            self.side = torch.cuda.Stream(device)   # the perimeter micro CTAs of a split step
            self.ev_prep = torch.cuda.Event()
            self.ev_side = torch.cuda.Event()
        self.peer_on = False

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.solver.device).cuda_stream)

    def pack(self, field, src):
        s = self.solver
        rc = s.lib.mm2d_halo_pack(s.ctx, field, C.c_void_p(0 if src is None else src.data_ptr()),
                                  self._stream())
        s._rc(rc)

    def unpack(self, field):
        s = self.solver
        s._rc(s.lib.mm2d_halo_unpack(s.ctx, field, self._stream()))

    def set_peers(self, neigh_G):
        """Peer form of the G halo (mm2d_halo_peer): ``neigh_G[s]`` is the
        current G tensor (or raw device pointer) of the neighbour in slot s,
        None for an inactive slot; ``None`` returns to the packed form."""
        s = self.solver
        self.peer_on = neigh_G is not None
        if neigh_G is None:
            s._rc(s.lib.mm2d_halo_peer(s.ctx, None))
            return
        ptrs = (C.c_void_p * 8)(*[None if t is None else
                                  (int(t) if isinstance(t, int) else t.data_ptr())
                                  for t in neigh_G])
        s._rc(s.lib.mm2d_halo_peer(s.ctx, ptrs))

    def phase(self, ph, Q, G, dt, Qout, Gout, H):
        s = self.solver
        from .solver import _ptr
        rc = s.lib.mm2d_step_phase(s.ctx, ph, _ptr(Q), _ptr(G), C.c_double(dt), _ptr(Qout),
                                   _ptr(Gout), _ptr(H), 0, None, None, None, self._stream())
        s._rc(rc)


def peer_views(blocks, states):
    """Per block, the current G tensors of its eight slot neighbours (all
    blocks held by this process, indexed by rank)."""
    return [[None if nb is None else states[nb][1] for nb in b.plan.slots] for b in blocks]


def _step_blocks_peer(blocks, exchange, states, dt, peers):
    """The decomposed step with the G halo in peer form: no G pack, transfer
    or receive buffer.  Each block's micro kernel (one launch, phase 0) reads
    its ghost cells in place from the neighbours' G^n arrays -- on another
    GPU through peer memory (NVLink), the perimeter CTAs' bulk copies
    fetching the halo rows while the interior CTAs compute.  The Q ring
    exchange that opens the step orders it against the neighbours: their
    sends follow their previous step on their streams, so once the ring has
    arrived their G^n is complete and their reads of this block's G^{n-1}
    buffer (which this step overwrites) are over."""
    import torch
    for b, st, nb in zip(blocks, states, peers):
        with torch.cuda.device(b.solver.device):
            b.set_peers(nb)
            b.pack(FIELD_Q, st[0])
    exchange.exchange(FIELD_Q)
    for b, st in zip(blocks, states):
        with torch.cuda.device(b.solver.device):
            b.unpack(FIELD_Q)
            b.phase(0, st[0], st[1], dt, st[2], st[3], st[4])
            b.pack(FIELD_H, None)
    exchange.exchange(FIELD_H)
    for b, st in zip(blocks, states):
        with torch.cuda.device(b.solver.device):
            b.unpack(FIELD_H)
            b.phase(1, st[0], st[1], dt, st[2], st[3], st[4])


class IpcPeers:
    """Peer form of the G halo with one process per GPU: this rank's two G
    buffers (the step's ping-pong) are cudaMalloc allocations whose CUDA-IPC
    handles every rank gathers; each rank maps its neighbours' buffers and
    passes the pair that holds their G^n to mm2d_halo_peer every step.  All
    ranks swap buffers together, so ``views(parity)`` of step n uses parity
    n % 2 on every rank."""

    def __init__(self, solver, plan: HaloPlan, shape, group=None):
        import torch
        import torch.distributed as dist
        self.lib, self.device, self.group = solver.lib, solver.device, group
        self.slots = plan.slots
        self.failed = None          # why the peer form is unavailable on this rank
        self.own, self.tensors, self.mapped = [], [], {}
        n = int(np.prod(shape))
        handles = []
        with torch.cuda.device(self.device):
            for _ in range(2):
                p, h = C.c_void_p(), C.create_string_buffer(64)
                if self.lib.mm2d_ipc_alloc(8 * n, C.byref(p), h) != 0:
                    self.failed = "mm2d_ipc_alloc failed"
                    break
                handles.append(h.raw)
                self.own.append(p.value)
            if self.failed is None:
                self.tensors = [torch.as_tensor(_CAI(p, n), device=self.device).view(shape)
                                for p in self.own]
        # (collective: every rank takes part, also one whose allocation failed)
        rank = dist.get_rank(group)
        gathered = [None] * dist.get_world_size(group)
        dist.all_gather_object(gathered, (rank, handles if self.failed is None else None),
                               group=group)
        table = dict(gathered)
        with torch.cuda.device(self.device):
            for nb in sorted({s for s in plan.slots if s is not None}):
                if self.failed is not None:
                    break
                if table[nb] is None:
                    self.failed = f"rank {nb} exported no buffers"
                    break
                ptrs = []
                for h in table[nb]:
                    p = C.c_void_p()
                    if self.lib.mm2d_ipc_open(h, C.byref(p)) != 0:
                        self.failed = f"mm2d_ipc_open failed for rank {nb}"
                        break
                    ptrs.append(p.value)
                self.mapped[nb] = ptrs

    def views(self, parity):
        return [None if nb is None else self.mapped[nb][parity] for nb in self.slots]

    def unmap(self):
        """Close this rank's mappings of its neighbours' buffers."""
        import torch
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            for ptrs in self.mapped.values():
                for p in ptrs:
                    self.lib.mm2d_ipc_close(C.c_void_p(p))
            self.mapped = {}

    def close(self, collective=True):
        """Collective: every rank unmaps its neighbours' buffers, then (after a
        barrier, so no importer still holds a mapping) frees its own.  With
        ``collective=False`` the caller provides that barrier (some ranks may
        hold no IpcPeers, e.g. after a failed mapping)."""
        import torch
        import torch.distributed as dist
        self.unmap()
        with torch.cuda.device(self.device):
            self.tensors = []
            if collective and dist.is_initialized():
                dist.barrier(group=self.group)
            for p in self.own:
                self.lib.mm2d_ipc_free(C.c_void_p(p))
            self.own = []


def step_blocks(blocks, exchange, states, dt, peers=None):
    """One decomposed step for every block held by this process.
    ``states[b] = (Q, G, Qout, Gout, H)`` device tensors of block b.
    ``peers`` (peer_views, or IPC mappings for one process per GPU) selects
    the peer form of the G halo (_step_blocks_peer); without it G travels
    packed:

    The G ring exchange (V doubles per perimeter cell, the bulk of the
    traffic) overlaps the interior cells' micro update: the Q ring (6
    doubles per cell) is exchanged first, then the G exchange is posted, the
    prep (phase 4) and every micro CTA that reads no received G halo (phase
    5) are enqueued, and only the perimeter CTAs (phase 3) wait for the G
    halo -- on a side stream that waits for the prep and the exchange, so
    they run concurrently with the interior CTAs instead of after them.
    Phases 4 + 5 + 3 are bitwise the unsplit phase 0."""
    import torch
    if peers is not None:
        return _step_blocks_peer(blocks, exchange, states, dt, peers)
    for b, st in zip(blocks, states):
        with torch.cuda.device(b.solver.device):
            if b.peer_on:
                b.set_peers(None)
            b.pack(FIELD_Q, st[0])
            b.pack(FIELD_G, st[1])
    exchange.exchange(FIELD_Q)
    hg = exchange.start(FIELD_G)
    for b, st in zip(blocks, states):
        with torch.cuda.device(b.solver.device):
            b.unpack(FIELD_Q)
            b.phase(4, st[0], st[1], dt, st[2], st[3], st[4])
            b.ev_prep.record()
            b.phase(5, st[0], st[1], dt, st[2], st[3], st[4])
    # the perimeter CTAs on each block's side stream, after its prep and the
    # G exchange (a stream-side wait over NCCL)
    for b in blocks:
        with torch.cuda.device(b.solver.device), torch.cuda.stream(b.side):
            b.side.wait_event(b.ev_prep)
            exchange.finish(hg)   # (a started exchange may be finished more than once)
    for b, st in zip(blocks, states):
        with torch.cuda.device(b.solver.device):
            with torch.cuda.stream(b.side):
                b.phase(3, st[0], st[1], dt, st[2], st[3], st[4])
                b.ev_side.record()
            torch.cuda.current_stream().wait_event(b.ev_side)
            b.pack(FIELD_H, None)
    exchange.exchange(FIELD_H)
    for b, st in zip(blocks, states):
        with torch.cuda.device(b.solver.device):
            b.unpack(FIELD_H)
            b.phase(1, st[0], st[1], dt, st[2], st[3], st[4])


class CapturedSteps:
    """The decomposed step of blocks that share one GPU, captured as two
    CUDA graphs (ping-pong between the (Q, G) and (Q_out, G_out) buffers of
    every block): a step is one graph launch instead of the ~8 C-ABI calls,
    halo copies and stream hand-offs per block that step_blocks issues from
    Python.  Replays are bitwise the eager step_blocks."""

    def __init__(self, blocks, exchange, states, dt, peer=False):
        import torch
        self.graphs = []
        dev = blocks[0].solver.device
        views = [states, [[st[2], st[3], st[0], st[1], st[4]] for st in states]]
        # (capturing records the work without running it: the states are
        # untouched until the first replay)
        with torch.cuda.device(dev):
            for v in views:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step_blocks(blocks, exchange, v, dt,
                                peers=peer_views(blocks, v) if peer else None)
                self.graphs.append(g)
        self.parity = 0

    def step(self):
        self.graphs[self.parity].replay()
        self.parity ^= 1


def enable_peer_access(blocks):
    """Peer access between the GPUs of neighbouring blocks (NVLink /
    NVSwitch); False if some pair cannot be mapped (the packed exchange is
    used then)."""
    ok = True
    lib = blocks[0].solver.lib
    for b in blocks:
        for nb in b.plan.slots:
            if nb is None:
                continue
            a, c = b.solver.device.index, blocks[nb].solver.device.index
            if a != c and lib.mm2d_enable_peer_access(a, c) != 0:
                ok = False
    return ok


def run_parallel_2d(mesh, bc, eps, model, Q0, G0, dt, n_steps, grid=(2, 2), track_from=None,
                    devices=None, graph=True, halo="peer"):
    """Advance n_steps with a rows x cols block grid spread over the visible
    GPUs (blocks round-robin over ``devices``); returns
    (Q, G, steady_max, seconds) like the reference (parallel.py:404-473).
    steady_max is the largest per-step max-norm change of Q over steps
    >= track_from (NaN if untracked); seconds is the wall time of the
    stepping loop (device-synchronised, excluding setup and gathers).

    When every block sits on one GPU and no steady-state tracking is asked
    for, the loop replays CUDA graphs of the decomposed step (``graph``);
    otherwise it is issued eagerly, ordered across GPUs by stream events
    only (no host synchronisation inside the loop).

    ``halo``: "peer" (default) reads the G ghost cells in place from the
    neighbour blocks' arrays (peer memory across GPUs; falls back to "packed"
    when a pair of GPUs has no peer access); "packed" packs, copies and
    receives the G ring, overlapped with the interior micro CTAs."""
    import torch
    nx, ny = mesh.space[0].n, mesh.space[1].n
    plans = make_plans(nx, ny, grid, bc)
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    blocks, states = [], []
    Q0 = np.asarray(Q0, dtype=np.float64)
    G0 = np.asarray(G0, dtype=np.float64)
    for p in plans:
        dev = torch.device("cuda", devices[p.rank % len(devices)])
        b = BlockStepper(mesh, bc, eps, model, grid, p, dev)
        blocks.append(b)
        Q = torch.from_numpy(np.ascontiguousarray(Q0[p.i0:p.i1, p.j0:p.j1])).to(dev)
        G = torch.from_numpy(np.ascontiguousarray(G0[p.i0:p.i1, p.j0:p.j1])).to(dev)
        H = torch.empty((4,) + p.shape, dtype=torch.float64, device=dev)
        states.append([Q, G, torch.empty_like(Q), torch.empty_like(G), H])
    exchange = LoopbackExchange(plans, [b.bufs for b in blocks])
    peer = halo == "peer" and enable_peer_access(blocks)
    steady = 0.0
    one_device = len({b.solver.device.index for b in blocks}) == 1
    captured = None
    if graph and one_device and track_from is None and n_steps >= 2:
        captured = CapturedSteps(blocks, exchange, states, dt, peer=peer)
    for d in devices:
        torch.cuda.synchronize(d)
    t0 = time.perf_counter()
    if captured is not None:
        with torch.cuda.device(blocks[0].solver.device):
            for n in range(n_steps):
                captured.step()
        if n_steps % 2:
            for st in states:
                st[0], st[2] = st[2], st[0]
                st[1], st[3] = st[3], st[1]
    else:
        for n in range(n_steps):
            step_blocks(blocks, exchange, states, dt,
                        peers=peer_views(blocks, states) if peer else None)
            if track_from is not None and n >= track_from:
                for st in states:
                    steady = max(steady, float((st[2] - st[0]).abs().max()))
            for st in states:
                st[0], st[2] = st[2], st[0]
                st[1], st[3] = st[3], st[1]
    for d in devices:
        torch.cuda.synchronize(d)
    seconds = time.perf_counter() - t0
    for b in blocks:
        b.solver.check()
    Q = np.empty_like(Q0)
    G = np.empty_like(G0)
    for p, st in zip(plans, states):
        Q[p.i0:p.i1, p.j0:p.j1] = st[0].cpu().numpy()
        G[p.i0:p.i1, p.j0:p.j1] = st[1].cpu().numpy()
    for b in blocks:
        b.solver.close()
    return Q, G, (steady if track_from is not None else float("nan")), seconds


__all__ = ["HaloPlan", "make_plans", "DistExchange", "LoopbackExchange", "BlockStepper",
           "halo_buffers", "step_blocks", "peer_views", "enable_peer_access", "IpcPeers",
           "CapturedSteps",
           "run_parallel_2d", "SLOTS", "OPPOSITE"]

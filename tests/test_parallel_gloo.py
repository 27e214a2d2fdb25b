"""Multi-rank logic of the block decomposition, on the CPU.

Plans follow the reference's numbering and neighbour wrap (pkg/tests/
test_parallel.py:47-71), and the slot exchange that runs over NCCL on the
GPUs is exercised here over gloo with world sizes 2 and 4: every rank packs
the edge cells of its block of a known global field (the C ABI's pack rule,
restated), exchanges, and must receive exactly the ghost cells the
reference's extract_ring would read from the global array
(parallel.py:109-150) on every exchanged face and corner.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_21832_b200.boundary import EXTRAPOLATE, PERIODIC, BoundarySpec2D, WallSpec
from paper_2509_21832_b200.errors import ConfigurationError
from paper_2509_21832_b200.parallel import OPPOSITE, DistExchange, make_plans

PERIODIC_BC = BoundarySpec2D(PERIODIC, PERIODIC, PERIODIC, PERIODIC)
MIXED_BC = BoundarySpec2D(EXTRAPOLATE, EXTRAPOLATE, PERIODIC, PERIODIC)
WALLS = BoundarySpec2D(WallSpec(1.0), WallSpec(1.0), WallSpec(1.0), WallSpec(1.0, 0.16))


def test_block_partition_and_numbering():
    plans = make_plans(12, 8, (3, 2), PERIODIC_BC)
    assert len(plans) == 6
    covered = np.zeros((12, 8), dtype=int)
    for p in plans:
        covered[p.i0:p.i1, p.j0:p.j1] += 1
        assert p.rank == p.pos[0] * 2 + p.pos[1]
    assert np.all(covered == 1)


def test_periodic_neighbours_wrap():
    plans = make_plans(8, 8, (2, 2), PERIODIC_BC)
    first = plans[0]
    assert first.neighbors["left"] == plans[2].rank
    assert first.neighbors["bottom"] == plans[1].rank
    # every face and corner is exchanged on a 2 x 2 periodic grid
    assert all(s is not None for s in first.slots)
    assert first.slots[4] == 3   # bottom-left corner wraps to block (1, 1)


def test_physical_faces_are_not_exchanged():
    plans = make_plans(8, 6, (2, 1), MIXED_BC)
    # x: extrapolate (physical) -> only the interior face; y: periodic over a
    # single block -> wrapped locally, no exchange
    assert plans[0].slots[:4] == (None, 1, None, None)
    assert plans[1].slots[:4] == (0, None, None, None)
    assert all(s is None for s in plans[0].slots[4:])
    w = make_plans(6, 6, (3, 3), WALLS)
    centre = w[4]
    assert all(s is not None for s in centre.slots)
    corner = w[0]
    assert corner.slots == (None, 3, None, 1, None, None, None, 4)


def test_grid_must_divide():
    with pytest.raises(ConfigurationError):
        make_plans(10, 8, (3, 2), PERIODIC_BC)


# -- gloo exchange ---------------------------------------------------------

def _slot_cells(p, s, ghost):
    """Global (i, j) of the edge (send) or ghost (receive) cells of slot s,
    in element order (the C ABI's slot_cell)."""
    bx, by = p.shape
    i0, j0 = p.i0, p.j0
    if s == 0:
        return [((i0 - 1) if ghost else i0, j0 + e) for e in range(by)]
    if s == 1:
        return [((i0 + bx) if ghost else (i0 + bx - 1), j0 + e) for e in range(by)]
    if s == 2:
        return [(i0 + e, (j0 - 1) if ghost else j0) for e in range(bx)]
    if s == 3:
        return [(i0 + e, (j0 + by) if ghost else (j0 + by - 1)) for e in range(bx)]
    di, dj = {4: (-1, -1), 5: (1, -1), 6: (-1, 1), 7: (1, 1)}[s]
    i = (i0 - 1 if di < 0 else i0 + bx) if ghost else (i0 if di < 0 else i0 + bx - 1)
    j = (j0 - 1 if dj < 0 else j0 + by) if ghost else (j0 if dj < 0 else j0 + by - 1)
    return [(i, j)]


def _worker(rank, world, port, nx, ny, grid, faces, width, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        bc = BoundarySpec2D(*faces)
        plans = make_plans(nx, ny, grid, bc)
        p = plans[rank]
        rng = np.random.default_rng(5)
        A = rng.standard_normal((nx, ny, width))
        bufs = [[(None, None)] * 8 for _ in range(3)]
        row = []
        for s in range(8):
            if p.slots[s] is None:
                row.append((None, None))
                continue
            cells = _slot_cells(p, s, ghost=False)
            send = torch.from_numpy(np.concatenate([A[i, j] for i, j in cells]))
            recv = torch.full((len(cells) * width,), np.nan, dtype=torch.float64)
            row.append((send, recv))
        bufs[1] = row
        # field 0 (the G ring in the step) carries -A and goes through the
        # split start / finish protocol step_blocks overlaps with compute
        bufs[0] = [(None, None) if sr[0] is None else (-sr[0], sr[1].clone()) for sr in row]
        ex = DistExchange(p, bufs)
        ex.exchange(1)
        h = ex.start(0)
        ex.finish(h)
        for f, sign in ((1, 1.0), (0, -1.0)):
            for s in range(8):
                if p.slots[s] is None:
                    continue
                ghosts = _slot_cells(p, s, ghost=True)
                want = sign * np.concatenate([A[i % nx, j % ny] for i, j in ghosts])
                got = bufs[f][s][1].numpy()
                if not np.array_equal(got, want):
                    errq.put(f"rank {rank} field {f} slot {s}: mismatch")
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        errq.put(f"rank {rank}: {exc!r}")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("grid,faces,shape", [
    ((2, 2), (PERIODIC,) * 4, (8, 6)),
    ((2, 1), (EXTRAPOLATE, EXTRAPOLATE, PERIODIC, PERIODIC), (8, 6)),
    ((1, 2), (PERIODIC, PERIODIC, WallSpec(1.0), WallSpec(1.0, 0.2)), (6, 8)),
    ((2, 2), (WallSpec(1.0),) * 4, (6, 8)),
])
def test_gloo_halo_exchange_matches_extract_ring(grid, faces, shape):
    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape[0], shape[1], grid, faces,
                                                6, errq)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    assert all(pr.exitcode == 0 for pr in procs), errors
    assert not errors, errors


def test_opposite_slots_are_involutions():
    assert all(OPPOSITE[OPPOSITE[s]] == s for s in range(8))


# -- step protocol ----------------------------------------------------------

def test_step_blocks_overlaps_g_exchange_with_interior_micro(monkeypatch):
    """step_blocks' order of operations (host logic, no GPU): the Q ring is
    exchanged first, the G exchange is posted and left in flight while the
    prep (phase 4) and the interior micro CTAs (phase 5) are enqueued, the
    perimeter CTAs (phase 3) go on the side stream after the prep and the G
    exchange, the main stream joins them, then the heat ring and the macro
    phase -- the reference worker grid's two barrier points
    (parallel.py:384-394) with the G transfer hidden behind interior work."""
    import contextlib
    from paper_2509_21832_b200 import parallel as par

    log = []
    monkeypatch.setattr(torch.cuda, "device", lambda d: contextlib.nullcontext())

    class Stream:
        def __init__(self, name):
            self.name = name

        def wait_event(self, ev):
            log.append(("wait", self.name, ev.name))

    class Event:
        def __init__(self, name):
            self.name = name

        def record(self):
            log.append(("record", self.name))

    cur = [Stream("main")]

    @contextlib.contextmanager
    def stream_ctx(st):
        prev, cur[0] = cur[0], st
        yield
        cur[0] = prev

    monkeypatch.setattr(torch.cuda, "stream", stream_ctx)
    monkeypatch.setattr(torch.cuda, "current_stream", lambda *a: cur[0])

    class Blk:
        side = Stream("side")
        ev_prep = Event("prep")
        ev_side = Event("side")
        peer_on = False

        def set_peers(self, nb):
            self.peer_on = nb is not None
            log.append(("peers", None if nb is None else tuple(nb)))

        class solver:
            device = torch.device("cpu")

        def pack(self, f, src):
            log.append(("pack", f))

        def unpack(self, f):
            log.append(("unpack", f))

        def phase(self, ph, *args):
            log.append(("phase", ph, cur[0].name))

    class Ex:
        def exchange(self, f):
            log.append(("exchange", f))

        def start(self, f):
            log.append(("start", f))
            return f

        def finish(self, h):
            log.append(("finish", h, cur[0].name))

    par.step_blocks([Blk()], Ex(), [(None,) * 5], 1e-3)
    G, Q, H = par.FIELD_G, par.FIELD_Q, par.FIELD_H
    assert log == [("pack", Q), ("pack", G), ("exchange", Q), ("start", G), ("unpack", Q),
                   ("phase", 4, "main"), ("record", "prep"), ("phase", 5, "main"),
                   ("wait", "side", "prep"), ("finish", G, "side"), ("phase", 3, "side"),
                   ("record", "side"), ("wait", "main", "side"), ("pack", H),
                   ("exchange", H), ("unpack", H), ("phase", 1, "main")]

    # peer form of the G halo: no G pack / exchange; the Q ring (which orders
    # the step against the neighbours) comes before the one micro launch
    # (phase 0) that reads the neighbours' arrays in place
    del log[:]
    blk = Blk()
    nb = [101, 102, None, None, None, None, None, None]
    par.step_blocks([blk], Ex(), [(None,) * 5], 1e-3, peers=[nb])
    assert log == [("peers", tuple(nb)), ("pack", Q), ("exchange", Q), ("unpack", Q),
                   ("phase", 0, "main"), ("pack", H), ("exchange", H), ("unpack", H),
                   ("phase", 1, "main")]
    # and a later packed step first returns the context to the packed form
    del log[:]
    par.step_blocks([blk], Ex(), [(None,) * 5], 1e-3)
    assert log[0] == ("peers", None) and log[1:3] == [("pack", Q), ("pack", G)]


def test_peer_views_follow_the_plans_slots():
    """peer_views: per block, the current G of the neighbour in each of the 8
    slots (None where the slot is a physical face or wraps locally)."""
    from paper_2509_21832_b200 import BoundarySpec2D, EXTRAPOLATE, PERIODIC
    from paper_2509_21832_b200.parallel import make_plans, peer_views
    from types import SimpleNamespace as NS
    plans = make_plans(8, 8, (2, 2), BoundarySpec2D(EXTRAPOLATE, EXTRAPOLATE, PERIODIC, PERIODIC))
    blocks = [NS(plan=p) for p in plans]
    states = [[None, f"G{p.rank}", None, None, None] for p in plans]
    views = peer_views(blocks, states)
    for p, v in zip(plans, views):
        assert v == [None if nb is None else f"G{nb}" for nb in p.slots]
    # rank 0 = block (0, 0): no left neighbour (extrapolate), right = rank 2,
    # bottom and top = rank 1 (periodic over two blocks in y)
    assert views[0][0] is None and views[0][1] == "G2" and views[0][2] == "G1" and views[0][3] == "G1"

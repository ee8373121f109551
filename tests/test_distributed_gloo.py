"""Slab decomposition (paper_2603_11868_b200/distributed.py) on CPU ranks
(gloo, world sizes 2 and 3): the multi-rank run must equal the single-process
reference restatement bit for bit -- every field by id, dt, nsub, interaction
and clamp counts -- through migrations, ghost refreshes and Shepard steps."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_11868_b200.distributed import (FIELDS, HALO_PLANES, SlabLayout,
                                               cell_plane)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(kind):
    from paper_2603_11868_b200 import cases
    if kind in ("tg2d", "tg3d"):
        # periodic Taylor-Green box with a uniform drift so
        # particles cross the wrap-around boundary between the end slabs
        d = 2 if kind == "tg2d" else 3
        cfg = cases.taylor_green_config(d, 40 if d == 2 else 16, precision="f32")
        reg, grid = cases.build_case(cfg)
        reg.raw_view("v")[:] += np.asarray([3.0, -2.0, 1.5][:d], np.float32)
        return reg, grid
    if kind == "2d":
        cfg = cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f32")
    else:
        cfg = cases.kleefsman_config(dp=0.08, precision="f32")
    return cases.build_case(cfg)


def _worker(rank, world, port, kind, steps, shepard_every, rebalance, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _dist_oracle_backend import OracleBackend
        from paper_2603_11868_b200.distributed import Comm, DistributedSimulation
        from paper_2603_11868_b200.physics import force_scalars
        reg, grid = _case(kind)
        n = reg.particle_count
        # arbitrary initial ownership: round-robin by id (first step migrates)
        sel = np.arange(n) % world == rank
        owned = {f: reg.raw_view(f)[sel] for f in FIELDS}
        sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
        be = OracleBackend(force_scalars(reg, grid), sing, grid)
        sim = DistributedSimulation(Comm(), be, grid, owned, sing,
                                    shepard_every=shepard_every,
                                    rebalance_every=rebalance)
        sim.initialize()
        rec = [(0.0, 0, sim.interaction_count, sim.out_of_bounds)]
        for _ in range(steps):
            dt = sim.advance()
            rec.append((dt, sim.last_nsub, sim.interaction_count, sim.out_of_bounds))
        g = sim.gather()
        stats = sim.comm.allreduce_i64([sim.migrated, sim.ghost_fluid])
        if rank == 0:
            out_q.put((rec, g, sim.layout.cuts.tolist(), stats.tolist()))
    finally:
        dist.destroy_process_group()


def _run(world, kind, steps, shepard_every=200, rebalance=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, kind, steps, shepard_every, rebalance, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _reference(kind, steps, shepard_every=200):
    from oracle.oracle import OracleSim
    reg, grid = _case(kind)
    sim = OracleSim.from_registry(reg, grid, shepard_every=shepard_every)
    sim.initialize()
    rec = [(0.0, 0, sim.interaction_count, sim.out_of_bounds)]
    for _ in range(steps):
        dt = sim.advance()
        rec.append((dt, sim.last_nsub, sim.interaction_count, sim.out_of_bounds))
    return rec, {f: sim.by_id(f) for f in FIELDS}


@pytest.mark.parametrize("world,kind,steps,shep,rebal", [
    (2, "2d", 60, 25, 10),
    (3, "2d", 40, 200, 1),
    (2, "3d", 6, 3, 2),
    (2, "tg2d", 40, 15, 5),
    (3, "tg2d", 30, 200, 1),
    (2, "tg3d", 8, 4, 2),
])
def test_slab_decomposition_matches_single_process(world, kind, steps, shep, rebal):
    rec, g, cuts, (migrated, ghosts) = _run(world, kind, steps, shep, rebal)
    assert migrated > 0 and ghosts > 0   # the exchanges were exercised
    ref_rec, ref = _reference(kind, steps, shep)
    assert rec == ref_rec
    for f in ("x", "v", "rho", "p", "m", "drho", "dvdt", "id", "wall", "nnb",
              "rho_scratch", "Vol"):
        assert g[f].tobytes() == ref[f].tobytes(), f


def test_slab_layout_balancing_and_halos():
    counts = np.array([0, 0, 5, 50, 50, 5, 0, 0, 10, 10, 0, 0], np.int64)
    lay = SlabLayout.balanced(counts, 3)
    assert lay.cuts[0] == 0 and lay.cuts[-1] == len(counts)
    assert (np.diff(lay.cuts) >= HALO_PLANES).all()
    owner = lay.owner(np.arange(len(counts)))
    for r in range(3):
        assert set(np.nonzero(owner == r)[0]) == set(range(lay.cuts[r], lay.cuts[r + 1]))
        halo = np.nonzero(lay.halo_mask(r, np.arange(len(counts))))[0]
        assert all((p < lay.cuts[r]) or (p >= lay.cuts[r + 1]) for p in halo)
        assert len(halo) <= 2 * HALO_PLANES
    with pytest.raises(ValueError):
        SlabLayout.balanced(np.ones(5), 3)


def test_periodic_ring_halos():
    """Axis-0 periodic layouts: halos wrap around the ring, never include the
    slab itself, and every plane within 2 of a slab (mod the ring) is in it."""
    P = 12
    lay = SlabLayout(np.array([0, 3, 8, 12], np.int64), P, True)
    planes = np.arange(P)
    for r in range(3):
        a, b = lay.cuts[r], lay.cuts[r + 1]
        halo = set(np.nonzero(lay.halo_mask(r, planes))[0])
        want = {(a - 1) % P, (a - 2) % P, b % P, (b + 1) % P} - set(range(a, b))
        assert halo == want, (r, halo, want)
    import torch
    t = lay.halo_mask(0, torch.arange(P))
    assert set(torch.nonzero(t).flatten().tolist()) == {10, 11, 3, 4}


def test_cell_plane_matches_kernel_binning():
    from oracle import oracle as O
    rng = np.random.default_rng(3)
    x = (rng.random((1000, 2)) * 3 - 0.5).astype(np.float32)
    origin = np.array([-0.14, -0.14], np.float32)
    shape = np.array([40, 30])
    keys, _ = O.compute_keys(x, origin, np.float32(0.065), shape)
    assert np.array_equal(cell_plane(x[:, 0], origin[0], np.float32(0.065), 40),
                          keys // 30)


class _RecordingComm:
    """Comm stand-in: records what each peer is sent and hands it back as
    that peer's message (a loopback), so packing and unpacking meet."""

    def __init__(self):
        import torch
        self.torch = torch
        self.device = torch.device("cpu")
        self.sent = {}

    def exchange(self, sends, recv_counts, row_shape, dtype):
        self.sent = {q: t.clone() for q, t in sends.items()}
        for q, t in sends.items():
            assert t.dtype == dtype and tuple(t.shape[1:]) == tuple(row_shape)
            assert t.shape[0] == recv_counts[q]
        return {q: t.clone() for q, t in sends.items()}


def test_exchange_fields_packs_only_the_sent_rows():
    """distributed.DistributedSimulation._exchange_fields: one int32 message
    per peer holding exactly the selected rows of every field, unpacked to
    the original dtypes and values; peers with no rows get no message."""
    import torch
    from paper_2603_11868_b200.distributed import DistributedSimulation
    rng = np.random.default_rng(5)
    n, d = 50, 3
    fields = {}
    for f in FIELDS:
        if f in ("x", "v", "dvdt"):
            fields[f] = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32))
        elif f in ("id", "wall", "nnb", "oflow"):
            fields[f] = torch.from_numpy(rng.integers(0, 1 << 30, n).astype(np.int32))
        else:
            fields[f] = torch.from_numpy(rng.standard_normal(n).astype(np.float32))
    sim = DistributedSimulation.__new__(DistributedSimulation)
    sim.comm = _RecordingComm()
    rows = {1: torch.tensor([3, 7, 7, 49]), 2: torch.tensor([0]),
            3: torch.zeros(0, dtype=torch.int64)}
    got = sim._exchange_fields(fields, rows, {1: 4, 2: 1, 3: 0})
    assert sorted(sim.comm.sent) == [1, 2]          # no empty message
    width = sum(3 if f in ("x", "v", "dvdt") else 1 for f in FIELDS)
    assert sim.comm.sent[1].shape == (4, width)
    for q in (1, 2):
        for f in FIELDS:
            assert got[f][q].dtype == fields[f].dtype
            assert torch.equal(got[f][q], fields[f][rows[q]])

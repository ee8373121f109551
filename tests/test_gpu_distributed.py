"""Slab decomposition with the CUDA engine as the per-rank compute
(distributed.EngineBackend): world sizes 2 and 3 as processes sharing the
box's one GPU, exchanging through gloo (host-staged, so no rank's kernel ever
waits on another's).  The multi-rank run must equal the single-process
reference restatement bit for bit -- every field by id, dt, nsub,
interaction and clamp counts -- through migrations, ghost refreshes, Shepard
steps and skin-list fix-ups."""

import os

import pytest
import torch.multiprocessing as mp

from test_distributed_gloo import _case, _free_port, _reference

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, kind, steps, shepard_every, rebalance, out_q):
    import numpy as np
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_11868_b200.distributed import (FIELDS, Comm, DistributedSimulation,
                                                       EngineBackend)
        from paper_2603_11868_b200.physics import force_scalars
        reg, grid = _case(kind)
        n = reg.particle_count
        sel = np.arange(n) % world == rank
        owned = {f: reg.raw_view(f)[sel] for f in FIELDS}
        sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
        be = EngineBackend(force_scalars(reg, grid), sing, grid, "cuda:0")
        sim = DistributedSimulation(Comm("cuda:0"), be, grid, owned, sing,
                                    shepard_every=shepard_every, rebalance_every=rebalance)
        sim.initialize()
        rec = [(0.0, 0, sim.interaction_count, sim.out_of_bounds)]
        for _ in range(steps):
            dt = sim.advance()
            rec.append((dt, sim.last_nsub, sim.interaction_count, sim.out_of_bounds))
        g = sim.gather()
        stats = sim.comm.allreduce_i64([sim.migrated, sim.ghost_fluid])
        if rank == 0:
            out_q.put((rec, g, stats.tolist()))
    finally:
        dist.destroy_process_group()


def _run(world, kind, steps, shepard_every, rebalance):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, kind, steps, shepard_every, rebalance, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,kind,steps,shep,rebal", [
    (2, "2d", 60, 25, 10),
    (3, "2d", 30, 200, 1),
    (2, "3d", 6, 3, 2),
    (2, "tg2d", 40, 15, 5),     # periodic ring of slabs
    (3, "tg3d", 8, 4, 2),
])
def test_engine_slabs_match_single_process(world, kind, steps, shep, rebal):
    rec, g, (migrated, ghosts) = _run(world, kind, steps, shep, rebal)
    assert migrated > 0 and ghosts > 0
    ref_rec, ref = _reference(kind, steps, shep)
    assert rec == ref_rec
    for f in ("x", "v", "rho", "p", "m", "drho", "dvdt", "id", "wall", "nnb",
              "rho_scratch", "Vol"):
        assert g[f].tobytes() == ref[f].tobytes(), f

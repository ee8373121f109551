"""Slab decomposition of the WCSPH step over ranks.

One process per GPU (``torch.distributed``; NCCL on GPUs, gloo for the CPU
tests).  The grid is cut along axis 0 into contiguous plane ranges (slabs);
a particle is owned by the rank whose slab contains the grid plane of its
position at the start of the advective step (its cell-linked-list plane).

Exactness argument.  The reference accumulates every neighbour sum in
ascending original id, so results do not depend on which process holds a
particle, only on each particle seeing exactly its reference neighbour set
with current values:

* a particle's neighbour block is the 3^d cell block around its CURRENT cell
  (neighborhood.py:188-213); within one advective step a particle moves less
  than one cell (dt_adv <= 0.25 h / vmax, cell = 2 h), so its current plane
  is within one plane of its start plane and its block within two planes of
  its slab: ghosts = particles whose start-of-step plane lies within
  ``HALO_PLANES = 2`` planes outside the slab (one plane is not enough);
* ghosts are refreshed from their owners exactly when the reference's data
  they carry changes: (x, v) after each drift, fluid (rho, p) after each
  density update, wall (rho, p) after each wall-pressure sweep, fluid
  (rho, p) after a Shepard filter;
* ghosts' own results are never read by owned particles, so computing them
  with a truncated neighbourhood is harmless (they are overwritten);
* time-step norms, stability inputs and counters are reduced over owned
  particles only (allreduce max / min / sum).

Hence an N-rank run is bit-identical to the 1-rank run and to the reference.

The per-rank compute is a backend: :class:`EngineBackend` (the CUDA engine,
below) in production, the CPU oracle composition in tests/.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

HALO_PLANES = 2

# per-particle state carried across ranks (registry field order)
FIELDS = ("x", "v", "rho", "p", "m", "Vol", "drho", "dvdt", "rho_scratch",
          "id", "wall", "nnb", "oflow")


def cell_plane(x0, origin0, cell_size, nplanes):
    """Axis-0 cell coordinate of positions, exactly as the kernels compute it
    (neighborhood.py:76-84: floor(f(f(x - o) / cs)), clamped)."""
    x0 = np.asarray(x0)
    dt = x0.dtype.type
    t = (x0 - dt(origin0)) / dt(cell_size)
    f = np.floor(t)
    with np.errstate(invalid="ignore"):
        c = np.where(~(f >= 0) | (f >= 9.2233720368547758e18), 0,
                     np.where(f < nplanes, f, nplanes - 1))
    return c.astype(np.int64)


@dataclass
class SlabLayout:
    """Plane cuts: rank r owns planes [cuts[r], cuts[r+1])."""
    cuts: np.ndarray
    nplanes: int

    @property
    def nranks(self):
        return len(self.cuts) - 1

    @staticmethod
    def even(nplanes, nranks):
        cuts = np.round(np.linspace(0, nplanes, nranks + 1)).astype(np.int64)
        return SlabLayout(cuts, nplanes)

    @staticmethod
    def balanced(plane_counts, nranks, min_width=HALO_PLANES):
        """Cuts that balance particle counts, every slab >= min_width planes
        so halos only ever come from adjacent ranks."""
        counts = np.asarray(plane_counts, np.int64)
        nplanes = counts.shape[0]
        if nplanes < nranks * min_width:
            raise ValueError(f"{nplanes} planes cannot hold {nranks} slabs of "
                             f">= {min_width} planes")
        cum = np.concatenate(([0], np.cumsum(counts)))
        total = cum[-1]
        cuts = [0]
        for r in range(1, nranks):
            target = total * r / nranks
            c = int(np.searchsorted(cum, target))
            lo = cuts[-1] + min_width
            hi = nplanes - (nranks - r) * min_width
            cuts.append(min(max(c, lo), hi))
        cuts.append(nplanes)
        return SlabLayout(np.asarray(cuts, np.int64), nplanes)

    def owner(self, planes):
        return np.searchsorted(self.cuts, np.asarray(planes), side="right") - 1

    def halo_mask(self, rank, planes):
        """Planes within HALO_PLANES outside rank's slab."""
        a, b = int(self.cuts[rank]), int(self.cuts[rank + 1])
        planes = np.asarray(planes)
        return ((planes >= a - HALO_PLANES) & (planes < a)) | \
               ((planes >= b) & (planes < b + HALO_PLANES))


class Comm:
    """Point-to-point and collective plumbing over torch.distributed."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        self.device = device if device is not None else torch.device("cpu")

    def _t(self, arr):
        torch = self.torch
        a = np.ascontiguousarray(arr)
        if a.dtype == np.uint32:
            a = a.view(np.int32)
        return torch.from_numpy(a).to(self.device)

    def allreduce(self, values, op):
        torch = self.torch
        t = torch.tensor(np.asarray(values, np.float64), device=self.device)
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX,
                                    "min": self.dist.ReduceOp.MIN,
                                    "sum": self.dist.ReduceOp.SUM}[op])
        return t.cpu().numpy()

    def allreduce_i64(self, values):
        torch = self.torch
        t = torch.tensor(np.asarray(values, np.int64), device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def exchange(self, sends, recv_counts, template):
        """sends: {rank: array}; recv_counts: {rank: n}; template gives the
        per-row shape / dtype.  Returns {rank: array} received."""
        torch = self.torch
        ops, recvs = [], {}
        row = template.shape[1:]
        dt = template.dtype
        tdt = np.int32 if dt == np.uint32 else dt
        for q, n in recv_counts.items():
            if n:
                buf = torch.empty((n,) + row, dtype=getattr(torch, np.dtype(tdt).name),
                                  device=self.device)
                recvs[q] = buf
                ops.append(self.dist.P2POp(self.dist.irecv, buf, q))
        sent = []
        for q, arr in sends.items():
            if len(arr):
                t = self._t(arr)
                sent.append(t)
                ops.append(self.dist.P2POp(self.dist.isend, t, q))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        out = {}
        for q, buf in recvs.items():
            a = buf.cpu().numpy()
            out[q] = a.view(np.uint32) if dt == np.uint32 else a
        return out

    def exchange_counts(self, counts):
        """All ranks' send counts: counts[q] = rows this rank sends to q;
        returns rows this rank receives from each q."""
        torch = self.torch
        send = torch.tensor([counts.get(q, 0) for q in range(self.size)],
                            dtype=torch.int64, device=self.device)
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send) if self.device.type != "cpu" \
            else self._alltoall_gloo(send, recv)
        return {q: int(recv[q].item()) for q in range(self.size) if q != self.rank}

    def _alltoall_gloo(self, send, recv):
        # gloo has no all_to_all_single; gather the matrix instead
        mats = [self.torch.empty_like(send) for _ in range(self.size)]
        self.dist.all_gather(mats, send)
        for q in range(self.size):
            recv[q] = mats[q][self.rank]


class DistributedSimulation:
    """Simulation.initialize/advance (physics.py:416-564) over slabs.

    ``owned``: dict of registry fields of the particles this rank owns at
    start (any partition is fine; the first step migrates).  ``backend``
    implements the per-rank phases on owned + ghost particles.
    """

    def __init__(self, comm, backend, grid, owned, sing, dt_max=1e-3, sort_every=100,
                 shepard_every=200, fixed_dt=None, cfl_acoustic=0.6,
                 cfl_advective=0.25, layout=None, rebalance_every=0):
        self.comm = comm
        self.backend = backend
        self.grid = grid
        self.owned = {f: np.array(owned[f], copy=True) for f in FIELDS}
        self.sing = sing
        self.dtype = self.owned["x"].dtype
        self.dt_max = dt_max
        self.sort_every = sort_every
        self.shepard_every = shepard_every
        self.fixed_dt = fixed_dt
        self.cfl_acoustic = cfl_acoustic
        self.cfl_advective = cfl_advective
        self.rebalance_every = rebalance_every
        nplanes = int(grid.shape[0])
        self.layout = layout or SlabLayout.even(nplanes, comm.size)
        self.step_count = 0
        self.time = 0.0
        self.interaction_count = 0
        self.out_of_bounds = 0
        self.last_nsub = 0
        self._send = {}        # rank -> local owned indices sent as ghosts
        self._ghost_from = {}  # rank -> (start, count) of its ghosts locally
        self._n_owned = 0
        self.migrated = 0      # particles sent to another rank (this rank)
        self.ghost_fluid = 0   # fluid ghosts received at the last step

    # -- decomposition ----------------------------------------------------------

    def _planes(self, x):
        return cell_plane(x[:, 0], self.grid.origin.astype(self.dtype)[0],
                          self.dtype.type(self.grid.cell_size), int(self.grid.shape[0]))

    def _rebalance(self):
        hist = np.bincount(self._planes(self.owned["x"]),
                           minlength=int(self.grid.shape[0]))
        tot = self.comm.allreduce_i64(hist)
        self.layout = SlabLayout.balanced(tot, self.comm.size)

    def _migrate(self):
        """Owned particles go to the owner of their current plane."""
        planes = self._planes(self.owned["x"])
        dest = self.layout.owner(planes)
        me = self.comm.rank
        keep = dest == me
        counts = {q: int((dest == q).sum()) for q in range(self.comm.size) if q != me}
        self.migrated += sum(counts.values())
        recv_counts = self.comm.exchange_counts(counts)
        new = {}
        for f in FIELDS:
            arr = self.owned[f]
            sends = {q: arr[dest == q] for q in counts}
            got = self.comm.exchange(sends, recv_counts, arr[:1] if len(arr) else
                                     np.zeros((1,) + arr.shape[1:], arr.dtype))
            parts = [arr[keep]] + [got[q] for q in sorted(got)]
            new[f] = np.concatenate(parts) if parts else arr[:0]
        # deterministic local order (by id) -- any order gives the same bits
        order = np.argsort(new["id"], kind="stable")
        self.owned = {f: new[f][order] for f in FIELDS}

    def _build_local(self):
        """Owned + ghosts; returns the local field dict and remembers the
        ghost send lists for the per-sub-step refreshes."""
        planes = self._planes(self.owned["x"])
        me = self.comm.rank
        self._send = {}
        for q in range(self.comm.size):
            if q == me:
                continue
            idx = np.nonzero(self.layout.halo_mask(q, planes))[0]
            if idx.size:
                self._send[q] = idx
        counts = {q: len(v) for q, v in self._send.items()}
        recv_counts = self.comm.exchange_counts(counts)
        n_own = len(self.owned["id"])
        local = {}
        self._ghost_from = {}
        off = n_own
        for q in sorted(recv_counts):
            self._ghost_from[q] = (off, recv_counts[q])
            off += recv_counts[q]
        for f in FIELDS:
            arr = self.owned[f]
            sends = {q: arr[idx] for q, idx in self._send.items()}
            got = self.comm.exchange(sends, recv_counts, arr[:1] if len(arr) else
                                     np.zeros((1,) + arr.shape[1:], arr.dtype))
            local[f] = np.concatenate([arr] + [got[q] for q in sorted(got)])
        self._n_owned = n_own
        self.ghost_fluid = int((local["wall"][n_own:] == 0).sum())
        return local

    def _refresh(self, names, walls):
        """Ghosts <- owners for fields ``names``; walls: None = all ghosts,
        False = fluid ghosts only, True = wall ghosts only."""
        wall_own = self.backend.get("wall", None)[: self._n_owned]
        sends = {}
        for q, idx in self._send.items():
            if walls is None:
                sel = idx
            elif walls:
                sel = idx[wall_own[idx] != 0]
            else:
                sel = idx[wall_own[idx] == 0]
            sends[q] = sel
        # receivers derive the same selection from the ghosts' own wall flags
        wall_loc = self.backend.get("wall", None)
        recv_sel = {}
        for q, (start, cnt) in self._ghost_from.items():
            g = np.arange(start, start + cnt)
            if walls is None:
                recv_sel[q] = g
            elif walls:
                recv_sel[q] = g[wall_loc[g] != 0]
            else:
                recv_sel[q] = g[wall_loc[g] == 0]
        for name in names:
            cur = self.backend.get(name, None)
            payload = {q: cur[sel] for q, sel in sends.items()}
            got = self.comm.exchange(payload, {q: len(s) for q, s in recv_sel.items()},
                                     cur[:1])
            for q, vals in got.items():
                self.backend.set(name, recv_sel[q], vals)

    # -- reference API ------------------------------------------------------------

    def _load_step(self):
        if self.rebalance_every and self.step_count % self.rebalance_every == 0:
            self._rebalance()
        self._migrate()
        local = self._build_local()
        oob = self.backend.load(local, self._n_owned, self.grid)
        self.out_of_bounds += int(self.comm.allreduce_i64([oob])[0])

    def initialize(self):
        self._load_step()
        self.backend.wall_pressure(initial=True)
        self._refresh(("rho", "p"), walls=True)
        self.backend.momentum_kick(None)
        self._finish_counts()

    def _finish_counts(self):
        inter, ovf = self.backend.counters()
        tot = self.comm.allreduce_i64([inter, ovf])
        if tot[1]:
            from .neighborhood import NeighborOverflowError, NEIGHBOR_CAPACITY
            raise NeighborOverflowError(
                f"neighbor buffer capacity {NEIGHBOR_CAPACITY} exceeded")
        self.interaction_count += int(tot[0])
        self.owned = self.backend.export_owned()

    def advance(self, end_time=None):
        from .physics import SimulationUnstableError, timestep_formula
        self._load_step()
        if self.shepard_every and self.step_count > 0 \
                and self.step_count % self.shepard_every == 0:
            self.backend.shepard()
            self._refresh(("rho", "p"), walls=False)
        vmax, amax = self.comm.allreduce(self.backend.norms(), "max")
        if self.fixed_dt is not None:
            dt_ac = dt_adv = self.fixed_dt
        else:
            dt_ac, dt_adv = timestep_formula(
                float(vmax), float(amax), float(self.sing["h"]), float(self.sing["c0"]),
                self.dt_max, self.cfl_acoustic, self.cfl_advective)
        dt = dt_adv
        if end_time is not None:
            dt = min(dt, end_time - self.time)
        nsub = max(1, int(math.ceil(dt / dt_ac)))
        dts = dt / nsub
        T = self.dtype.type
        half, full = T(0.5 * dts), T(dts)
        for _ in range(nsub):
            self.backend.kick_drift(half, full)
            self._refresh(("x", "v"), walls=False)
            self.backend.continuity_du(full)
            self._refresh(("rho", "p"), walls=False)
            self.backend.wall_pressure()
            self._refresh(("rho", "p"), walls=True)
            self.backend.momentum_kick(half)
        self.last_nsub = nsub
        self._finish_counts()
        self.step_count += 1
        self.time += dt
        rho_min, v2 = self.backend.stability()
        rho_min = float(self.comm.allreduce([rho_min], "min")[0])
        v2 = float(self.comm.allreduce([v2], "max")[0])
        c0 = float(self.sing["c0"])
        if rho_min <= 0.0:
            raise SimulationUnstableError(f"non-positive density at step {self.step_count}")
        if float(np.sqrt(self.dtype.type(v2))) > 10.0 * c0:
            raise SimulationUnstableError(f"runaway velocity at step {self.step_count}")
        return dt

    def gather(self):
        """All owned particles of all ranks, ordered by id (every rank)."""
        out = {}
        for f in FIELDS:
            lst = [None] * self.comm.size
            self.comm.dist.all_gather_object(lst, self.owned[f])
            out[f] = np.concatenate(lst)
        order = np.argsort(out["id"], kind="stable")
        return {f: out[f][order] for f in FIELDS}

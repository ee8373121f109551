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

Data plane.  Per-particle state lives in torch tensors on the rank's device
(uint32 fields as int32); migration and ghost exchange are
``batch_isend_irecv`` between neighbouring ranks -- NCCL moves device memory
directly, gloo (CPU tests) stages through the host.  The per-rank compute is
a backend: :class:`EngineBackend` (the CUDA engine, device-resident) in
production, the CPU oracle composition in tests/.  Backends own the halo
record format (``pack`` / ``unpack``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

HALO_PLANES = 2
SLAB_MAX_PEERS = 8     # include/sph_b200.h SPH_MAX_PEERS

# per-particle state carried across ranks (registry field order)
FIELDS = ("x", "v", "rho", "p", "m", "Vol", "drho", "dvdt", "rho_scratch",
          "id", "wall", "nnb", "oflow")
INDEX_FIELDS = ("id", "wall", "nnb", "oflow")

# halo record kinds (include/sph_b200.h SPH_HALO_*)
XV, RP_NEXT, RP_CUR = 0, 1, 2


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


def _torch():
    import torch
    return torch


def as_tensor(arr, device):
    """numpy field -> torch tensor on device (uint32 as int32)."""
    torch = _torch()
    if isinstance(arr, torch.Tensor):
        return arr.to(device)
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device)


def to_numpy(t, name):
    a = t.detach().cpu().numpy()
    return a.view(np.uint32) if name in INDEX_FIELDS else a


@dataclass
class SlabLayout:
    """Plane cuts: rank r owns planes [cuts[r], cuts[r+1])."""
    cuts: np.ndarray
    nplanes: int
    # axis 0 periodic: the slabs form a ring and halos
    # wrap around plane 0 / nplanes - 1
    periodic: bool = False

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
        """Owning rank of each plane (numpy or torch input, same kind out)."""
        torch = _torch()
        if isinstance(planes, torch.Tensor):
            cuts = torch.as_tensor(self.cuts, device=planes.device)
            return torch.searchsorted(cuts, planes, right=True) - 1
        return np.searchsorted(self.cuts, np.asarray(planes), side="right") - 1

    def halo_mask(self, rank, planes):
        """Planes within HALO_PLANES outside rank's slab."""
        a, b = int(self.cuts[rank]), int(self.cuts[rank + 1])
        if self.periodic:
            # distance outside the slab measured around the ring
            P = self.nplanes
            below = (a - planes) % P      # 1, 2: just below a (wrapping)
            above = (planes - b) % P      # 0, 1: at or just above b (wrapping)
            inside = (planes >= a) & (planes < b)
            return ~inside & (((below >= 1) & (below <= HALO_PLANES)) |
                              (above < HALO_PLANES))
        return ((planes >= a - HALO_PLANES) & (planes < a)) | \
               ((planes >= b) & (planes < b + HALO_PLANES))


class Comm:
    """Point-to-point and collective plumbing over torch.distributed.

    ``device``: where the data plane lives.  NCCL moves device tensors
    directly; gloo only moves host tensors, so device tensors are staged."""

    def __init__(self, device=None):
        torch = _torch()
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.gloo = dist.get_backend() == "gloo"
        self.wire = torch.device("cpu") if self.gloo else self.device

    def allreduce(self, values, op):
        t = self.torch.tensor(np.asarray(values, np.float64), device=self.wire)
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX,
                                    "min": self.dist.ReduceOp.MIN,
                                    "sum": self.dist.ReduceOp.SUM}[op])
        return t.cpu().numpy()

    def allreduce_i64(self, values):
        t = self.torch.tensor(np.asarray(values, np.int64), device=self.wire)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy()

    def exchange(self, sends, recv_counts, row_shape, dtype):
        """sends: {rank: tensor (k, *row_shape)}; recv_counts: {rank: n}.
        Returns {rank: tensor} received, on self.device."""
        torch = self.torch
        ops, recvs, keep = [], {}, []
        for q, n in recv_counts.items():
            if n:
                buf = torch.empty((n,) + tuple(row_shape), dtype=dtype, device=self.wire)
                recvs[q] = buf
                ops.append(self.dist.P2POp(self.dist.irecv, buf, q))
        for q, t in sends.items():
            if t.shape[0]:
                t = t.contiguous().to(self.wire)
                keep.append(t)
                ops.append(self.dist.P2POp(self.dist.isend, t, q))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return {q: b.to(self.device) for q, b in recvs.items()}

    def exchange_counts(self, counts, width=None):
        """All ranks' send counts: counts[q] = rows this rank sends to q
        (or a tuple of `width` counts); returns what this rank receives from
        each q (ints, or lists of `width`)."""
        torch = self.torch
        w = width or 1
        rows = [counts.get(q, 0 if width is None else (0,) * w) for q in range(self.size)]
        send = torch.tensor(rows if width else [[c] for c in rows],
                            dtype=torch.int64, device=self.wire).reshape(-1)
        if self.gloo:   # gloo has no all_to_all_single: gather the matrix
            mats = [torch.empty_like(send) for _ in range(self.size)]
            self.dist.all_gather(mats, send)
            recv = torch.stack([m.view(self.size, w)[self.rank] for m in mats])
        else:
            recv = torch.empty_like(send)
            self.dist.all_to_all_single(recv, send)
            recv = recv.view(self.size, w)
        recv = recv.cpu().tolist()
        return {q: (recv[q] if width else int(recv[q][0]))
                for q in range(self.size) if q != self.rank}


class DistributedSimulation:
    """Simulation.initialize/advance (physics.py:416-564) over slabs.

    ``owned``: dict of registry fields (numpy or torch) of the particles this
    rank owns at start (any partition is fine; the first step migrates).
    ``backend`` runs the per-rank phases on owned + ghost particles.
    """

    def __init__(self, comm, backend, grid, owned, sing, dt_max=1e-3, sort_every=100,
                 shepard_every=200, fixed_dt=None, cfl_acoustic=0.6,
                 cfl_advective=0.25, layout=None, rebalance_every=0):
        self.comm = comm
        self.backend = backend
        self.grid = grid
        self.owned = {f: as_tensor(owned[f], comm.device).clone() for f in FIELDS}
        self.sing = sing
        self.dtype = np.dtype(str(self.owned["x"].dtype).replace("torch.", ""))
        self.dt_max = dt_max
        self.sort_every = sort_every      # physical order is per rank; not mirrored
        self.shepard_every = shepard_every
        self.fixed_dt = fixed_dt
        self.cfl_acoustic = cfl_acoustic
        self.cfl_advective = cfl_advective
        self.rebalance_every = rebalance_every
        nplanes = int(grid.shape[0])
        per = getattr(grid, "period", None)
        self._periodic0 = per is not None and float(per[0]) > 0.0
        self.layout = self._ring(layout or SlabLayout.even(nplanes, comm.size))
        self.step_count = 0
        self.time = 0.0
        self.interaction_count = 0
        self.out_of_bounds = 0
        self.last_nsub = 0
        self._sel = {}         # "fluid"/"wall" -> (send rows {q}, ghost rows {q})
        self._n_owned = 0
        self.migrated = 0      # particles sent to another rank (this rank)
        self._layout_seen = None   # layout of the last device migration
        self.ghost_fluid = 0   # fluid ghosts received at the last step
        if hasattr(backend, "attach"):
            backend.attach(comm)
        if hasattr(backend, "set_id_range"):   # global ids are 0 .. N-1
            backend.set_id_range(int(comm.allreduce_i64([int(self.owned["id"].shape[0])])[0]))

    # -- decomposition ----------------------------------------------------------

    def _ring(self, layout):
        """The layout as a ring of slabs when axis 0 is periodic."""
        if self._periodic0 and not layout.periodic:
            return SlabLayout(layout.cuts, layout.nplanes, True)
        return layout

    def _planes(self, x):
        return self.backend.planes(x)

    def _rebalance(self):
        torch = self.comm.torch
        planes = self._planes(self.owned["x"])
        hist = torch.bincount(planes, minlength=int(self.grid.shape[0])).cpu().numpy()
        tot = self.comm.allreduce_i64(hist)
        self.layout = self._ring(SlabLayout.balanced(tot, self.comm.size))

    def _exchange_fields(self, fields, send_rows, recv_counts):
        """Rows of every field to each neighbour in ONE message: the fields
        are viewed as int32 columns of one (n, width) matrix."""
        torch = self.comm.torch
        widths = [int(np.prod(fields[f].shape[1:], dtype=np.int64)) *
                  fields[f].element_size() // 4 for f in FIELDS]

        def pack(rows):   # only the rows sent: the halo, not the whole rank
            k = int(rows.numel())
            return torch.cat([fields[f].index_select(0, rows).reshape(k, -1).view(torch.int32)
                              for f in FIELDS], dim=1)

        got = self.comm.exchange({q: pack(r) for q, r in send_rows.items() if r.numel()},
                                 recv_counts, (sum(widths),), torch.int32)
        out = {f: {} for f in FIELDS}
        for q, m in got.items():
            c0 = 0
            for f, w in zip(FIELDS, widths):
                ref = fields[f]
                out[f][q] = m[:, c0:c0 + w].contiguous().view(ref.dtype).reshape(
                    (m.shape[0],) + tuple(ref.shape[1:]))
                c0 += w
        return out

    def _migrate(self):
        """Owned particles go to the owner of their current plane."""
        torch = self.comm.torch
        me = self.comm.rank
        dest = self.layout.owner(self._planes(self.owned["x"]))
        keep = dest == me
        # per-rank counts as W reductions (a CUDA bincount into W bins
        # serialises on a few global atomics)
        cnt = torch.stack([(dest == q).sum() for q in range(self.comm.size)]).cpu().tolist()
        send_rows = {q: torch.nonzero(dest == q).flatten()
                     for q in range(self.comm.size) if q != me and cnt[q]}
        self.migrated += sum(cnt[q] for q in send_rows)
        recv_counts = self.comm.exchange_counts({q: cnt[q] for q in send_rows})
        got = self._exchange_fields(self.owned, send_rows, recv_counts)
        # any local order gives the same bits (sums run in id order); kept
        # particles first, then arrivals by source rank
        if send_rows or any(got[f] for f in ("id",)):
            kept = torch.nonzero(keep).flatten()
            self.owned = {f: torch.cat([self.owned[f].index_select(0, kept)] +
                                       [got[f][q] for q in sorted(got[f])]) for f in FIELDS}

    def _build_local(self):
        """Owned + ghosts (rows [0, n_own) owned, then ghosts grouped by
        source rank); remembers the send/receive rows of the refreshes."""
        torch = self.comm.torch
        me = self.comm.rank
        planes = self._planes(self.owned["x"])
        send_rows = {}
        for q in range(self.comm.size):
            if q == me:
                continue
            idx = torch.nonzero(self.layout.halo_mask(q, planes)).flatten()
            if idx.numel():
                send_rows[q] = idx
        recv_counts = self.comm.exchange_counts({q: len(v) for q, v in send_rows.items()})
        got = self._exchange_fields(self.owned, send_rows, recv_counts)
        n_own = int(self.owned["id"].shape[0])
        local = {f: torch.cat([self.owned[f]] + [got[f][q] for q in sorted(got[f])])
                 if got[f] else self.owned[f] for f in FIELDS}
        ghost_rows, off = {}, n_own
        for q in sorted(recv_counts):
            ghost_rows[q] = torch.arange(off, off + recv_counts[q], device=self.comm.device)
            off += recv_counts[q]
        wall = local["wall"]
        self._sel = {}
        for name, want_wall in (("fluid", False), ("wall", True)):
            s = {q: r[(wall[r] != 0) == want_wall] for q, r in send_rows.items()}
            g = {q: r[(wall[r] != 0) == want_wall] for q, r in ghost_rows.items()}
            self._sel[name] = (s, g)
        self._n_owned = n_own
        self.ghost_fluid = int((wall[n_own:] == 0).sum())
        return local

    def _refresh(self, kind, which):
        """Ghosts <- owners: halo records of `kind` for the fluid or wall
        ghosts (`which`)."""
        send_rows, ghost_rows = self._sel[which]
        be = self.backend
        if hasattr(be, "halo_pack"):   # backend-packed buffers (engine)
            payload = be.halo_pack(kind, which)
            got = self.comm.exchange(payload,
                                     {q: int(r.numel()) for q, r in ghost_rows.items()},
                                     (be.halo_width(kind),), be.halo_dtype)
            be.halo_unpack(kind, which, got)
            return
        payload = {q: be.pack(kind, r) for q, r in send_rows.items()}
        got = self.comm.exchange(payload, {q: int(r.numel()) for q, r in ghost_rows.items()},
                                 (be.halo_width(kind),), be.halo_dtype)
        for q, buf in got.items():
            be.unpack(kind, ghost_rows[q], buf)

    # -- reference API ------------------------------------------------------------

    def _peers(self):
        """The ranks this rank exchanges with: its axis-0 neighbours (a ring
        when axis 0 is periodic; one peer when both neighbours coincide)."""
        me, W = self.comm.rank, self.comm.size
        if W == 1:
            return []
        if self.layout.periodic:
            return sorted({(me - 1) % W, (me + 1) % W})
        return [q for q in (me - 1, me + 1) if 0 <= q < W]

    def _classify(self, fields, peers):
        """Device classification of the owned rows (csrc/slab.cu): per peer
        mover / fluid-halo / wall-halo row lists, the kept rows, and the
        out-of-bounds count, with ONE device->host read of the counts."""
        lists, cnt = self.backend.classify(fields, self.layout, self.comm.rank, peers)
        P = len(peers)
        if cnt[3 * P + 1]:
            raise RuntimeError("a particle crossed more than one slab in one step")
        return peers, lists, cnt

    def _load_step_device(self):
        """_migrate + _build_local on the device: classification, record
        packing and row assembly are library kernels; the host sees two count
        vectors per step (one per exchange round)."""
        be = self.backend
        torch = self.comm.torch
        # round 1: movers (classified on the step-start positions).  A step
        # moves a particle by less than a plane, so movers go to neighbours --
        # except at the first step (any initial partition) and after a
        # re-cut, when any rank may be the new owner
        W, me = self.comm.size, self.comm.rank
        everyone = [q for q in range(W) if q != me]
        anywhere = (self._layout_seen is not self.layout) and len(everyone) <= SLAB_MAX_PEERS
        self._layout_seen = self.layout
        peers, lists, cnt = self._classify(self.owned, everyone if anywhere else self._peers())
        P = len(peers)
        oob = int(cnt[3 * P + 2])
        sends = {q: be.pack_rows(self.owned, lists[3 * k], int(cnt[3 * k]))
                 for k, q in enumerate(peers) if cnt[3 * k]}
        got = self.comm.exchange(sends, self.comm.exchange_counts(
            {q: int(cnt[3 * k]) for k, q in enumerate(peers)}), (be.record_words,), torch.int32)
        self.migrated += sum(int(cnt[3 * k]) for k in range(P))
        n_keep = int(cnt[3 * P])
        if sends or got:
            arr = [got[q] for q in sorted(got)]
            owned = be.empty_rows(n_keep + sum(int(a.shape[0]) for a in arr))
            be.gather_rows(self.owned, lists[3 * P], n_keep, owned, 0)
            off = n_keep
            for a in arr:
                be.unpack_rows(a, owned, off)
                off += int(a.shape[0])
            self.owned = owned
        # round 2: halos of the post-migration owned set (fluid records first)
        peers, lists, cnt = self._classify(self.owned, self._peers())
        n_own = int(self.owned["id"].shape[0])
        sends, scount = {}, {}
        for k, q in enumerate(peers):
            nf, nw = int(cnt[3 * k + 1]), int(cnt[3 * k + 2])
            scount[q] = (nf, nw)
            if nf + nw:
                rec = torch.empty((nf + nw, be.record_words), dtype=torch.int32,
                                  device=self.comm.device)
                be.pack_rows(self.owned, lists[3 * k + 1], nf, rec[:nf])
                be.pack_rows(self.owned, lists[3 * k + 2], nw, rec[nf:])
                sends[q] = rec
        rcount = self.comm.exchange_counts(scount, width=2)
        got = self.comm.exchange(sends, {q: sum(c) for q, c in rcount.items()},
                                 (be.record_words,), torch.int32)
        n_ghost = sum(sum(c) for c in rcount.values())
        local = be.empty_rows(n_own + n_ghost)
        be.copy_rows(self.owned, local, n_own)
        sel_f, sel_w, off = ({}, {}), ({}, {}), n_own
        dev = self.comm.device
        for k, q in enumerate(peers):
            nf, nw = scount[q]
            if nf:
                sel_f[0][q] = lists[3 * k + 1][:nf].to(torch.int64)
            if nw:
                sel_w[0][q] = lists[3 * k + 2][:nw].to(torch.int64)
        for q in sorted(rcount):
            gf, gw = rcount[q]
            if gf + gw:
                be.unpack_rows(got[q], local, off)
            if gf:
                sel_f[1][q] = torch.arange(off, off + gf, device=dev)
            if gw:
                sel_w[1][q] = torch.arange(off + gf, off + gf + gw, device=dev)
            off += gf + gw
        self._sel = {"fluid": sel_f, "wall": sel_w}
        self._n_owned = n_own
        self.ghost_fluid = sum(c[0] for c in rcount.values())
        be.load(local, n_own, self.grid, count_oob=False)
        if hasattr(be, "set_halo"):
            be.set_halo(self._sel)
        self.out_of_bounds += int(self.comm.allreduce_i64([oob])[0])

    def _load_step(self):
        if self.rebalance_every and self.step_count % self.rebalance_every == 0:
            self._rebalance()
        if getattr(self.backend, "device_rows", False):
            self._load_step_device()
            return
        self._migrate()
        local = self._build_local()
        oob = self.backend.load(local, self._n_owned, self.grid)
        if hasattr(self.backend, "set_halo"):
            self.backend.set_halo(self._sel)
        self.out_of_bounds += int(self.comm.allreduce_i64([oob])[0])

    def initialize(self):
        self._load_step()
        self.backend.prepare(None)
        self.backend.wall_pressure(initial=True)
        self._refresh(RP_CUR, "wall")
        self.backend.momentum_kick(None)
        self._finish_counts()

    def _finish_counts(self):
        inter, ovf = self.backend.counters()
        tot = [inter, ovf] if getattr(self.backend, "global_stats", False) else \
            self.comm.allreduce_i64([inter, ovf])
        if tot[1]:
            from .neighborhood import NeighborOverflowError, NEIGHBOR_CAPACITY
            raise NeighborOverflowError(
                f"neighbor buffer capacity {NEIGHBOR_CAPACITY} exceeded")
        self.interaction_count += int(tot[0])
        self.owned = self.backend.export_owned()

    def advance(self, end_time=None):
        from .physics import SimulationUnstableError, timestep_formula
        self._load_step()
        # compute_timestep reads only v and dvdt, which Shepard leaves alone
        norms = self.backend.norms()
        vmax, amax = norms if getattr(self.backend, "global_stats", False) else \
            self.comm.allreduce(norms, "max")
        if self.fixed_dt is not None:
            dt_ac = dt_adv = self.fixed_dt
        else:
            dt_ac, dt_adv = timestep_formula(
                float(vmax), float(amax), float(self.sing["h"]), float(self.sing["c0"]),
                self.dt_max, self.cfl_acoustic, self.cfl_advective)
        dt = dt_adv
        if end_time is not None:
            dt = min(dt, end_time - self.time)
        self.backend.prepare((float(vmax), float(amax), dt))
        if self.shepard_every and self.step_count > 0 \
                and self.step_count % self.shepard_every == 0:
            self.backend.shepard()
            self._refresh(RP_CUR, "fluid")
        nsub = max(1, int(math.ceil(dt / dt_ac)))
        dts = dt / nsub
        T = self.dtype.type
        half, full = T(0.5 * dts), T(dts)
        if getattr(self.backend, "native_loop", False):
            # the engine enqueues the sub-steps with their NCCL refreshes itself
            self.backend.substeps(half, full, nsub)
        else:
            for k in range(nsub):
                self.backend.kick_drift(half, full)
                self._refresh(XV, "fluid")
                self.backend.continuity_du(full)
                self._refresh(RP_NEXT, "fluid")
                self.backend.wall_pressure()
                self._refresh(RP_NEXT, "wall")
                # the next sub-step's kick + drift may be fused into this sweep
                self.backend.momentum_kick(half, full if k + 1 < nsub else None)
        self.last_nsub = nsub
        self._finish_counts()
        self.step_count += 1
        self.time += dt
        rho_min, v2 = self.backend.stability()
        if not getattr(self.backend, "global_stats", False):
            rho_min = float(self.comm.allreduce([rho_min], "min")[0])
            v2 = float(self.comm.allreduce([v2], "max")[0])
        c0 = float(self.sing["c0"])
        if rho_min <= 0.0:
            raise SimulationUnstableError(f"non-positive density at step {self.step_count}")
        if float(np.sqrt(self.dtype.type(v2))) > 10.0 * c0:
            raise SimulationUnstableError(f"runaway velocity at step {self.step_count}")
        return dt

    def checkpoint(self):
        """The rank's state between steps (owned particles, layout, counters):
        restore() repeats the following steps bit for bit."""
        be = self.backend
        return ({f: t.clone() for f, t in self.owned.items()}, self.layout,
                {k: getattr(self, k) for k in ("step_count", "time", "interaction_count",
                                               "out_of_bounds", "migrated")},
                getattr(be, "_skin_factor", None))

    def restore(self, ck):
        owned, layout, attrs, skin = ck
        self.owned = {f: t.clone() for f, t in owned.items()}
        self.layout = layout
        for k, v in attrs.items():
            setattr(self, k, v)
        if skin is not None:
            self.backend._skin_factor = skin

    def gather(self):
        """All owned particles of all ranks as numpy, ordered by id (every rank)."""
        out = {}
        for f in FIELDS:
            lst = [None] * self.comm.size
            self.comm.dist.all_gather_object(lst, to_numpy(self.owned[f], f))
            out[f] = np.concatenate(lst)
        order = np.argsort(out["id"], kind="stable")
        return {f: out[f][order] for f in FIELDS}


class EngineBackend:
    """The CUDA engine (csrc/engine.cu) as the per-rank compute of a slab.

    Each step the rank's owned + ghost particles are pushed (device to
    device) into one engine with local ids = rank of the global id (the
    accumulation order is therefore the reference's), ghosts flagged in
    ``owned_id`` so they are neither integrated nor counted; the phases run
    through ``sph_engine_phase`` and halo records through
    ``sph_engine_pack/unpack`` at physical indices.
    """

    def __init__(self, scalars, sing, grid, device):
        torch = _torch()
        from . import _native
        from .physics import grid_is_periodic
        self.L = _native.lib(periodic=grid_is_periodic(grid))
        self._native = _native
        self.scalars = scalars
        self.sing = sing
        self.grid = grid
        self.device = torch.device(device)
        self.f64 = np.dtype(type(scalars[0])) == np.float64
        self.np_dtype = np.float64 if self.f64 else np.float32
        self.halo_dtype = torch.float64 if self.f64 else torch.float32
        self.dim = grid.dim
        self.E = None
        self.T = None
        self._caps = (0, 0, 0)
        self.id_range = 0         # > 0: the engine runs on GLOBAL ids (set_id_range)
        self._skin_factor = 3.0
        self.comm_handle = None     # NCCL communicator of the library (NCCL runs)
        self.native_loop = False
        self.plan = None
        from ._device import stream_ptr
        self.stream = stream_ptr(self.device)

    # -- helpers ------------------------------------------------------------------

    def _call(self, name, *args):
        rc = getattr(self.L, name)(ctypes.byref(self.E), *args, self.stream)
        self._native.check(rc, name)

    def _stats(self):
        torch = _torch()
        host = self.T["stats"].cpu()
        torch.cuda.current_stream(self.device).synchronize()
        return self._native.SphStepStats.from_buffer_copy(host.numpy().tobytes())

    def set_id_range(self, n_total):
        """Ids are the global registry ids 0 .. n_total-1: the engine's by-id
        arrays span them, so no per-step local relabelling is needed."""
        self.id_range = int(n_total)

    def _ensure(self, n, nf, nw):
        from .physics import engine_alloc, engine_set_counts
        cn, cf, cw = self._caps
        if self.E is None or n > cn or nf > cf or nw > cw:
            grow = lambda a, c: max(a, int(c * 1.15) + 64)   # noqa: E731
            caps = (grow(n, cn), grow(nf, cf), grow(nw, cw))
            # slab engines re-push every step: no persistent-list buffers
            self.E, self.T = engine_alloc(self.device, caps[0], caps[1], caps[2], self.dim,
                                          self.f64, self.grid, self.scalars, self.sing["g"],
                                          id_range=self.id_range, persist=False)
            self._caps = caps
        engine_set_counts(self.E, n, nf)
        self.E.owned_id = self.T["owned_id"].data_ptr()

    def planes(self, x):
        """Axis-0 cell planes of positions x (n, d) on the device, by the
        library's binning kernel (neighborhood.py:76-84)."""
        torch = _torch()
        n = int(x.shape[0])
        if n == 0:
            return torch.zeros(0, dtype=torch.int64, device=self.device)
        keys, _ = self._keys(x)
        per_plane = int(np.prod(self.grid.shape[1:]))
        return keys // per_plane

    def _keys(self, x):
        torch = _torch()
        n = int(x.shape[0])
        keys = torch.empty(n, dtype=torch.int64, device=self.device)
        oob = torch.zeros(1, dtype=torch.int32, device=self.device)
        origin = np.zeros(3, self.np_dtype)
        origin[:self.dim] = self.grid.origin.astype(self.np_dtype)
        shape = np.ones(3, np.int64)
        shape[:self.dim] = self.grid.shape
        fn = getattr(self.L, f"sph_cell_keys_{self._native.sfx(np.dtype(self.np_dtype))}")
        xc = x.contiguous()
        rc = fn(ctypes.c_void_p(xc.data_ptr()), n, self.dim,
                origin.ctypes.data_as(ctypes.c_void_p), self.np_dtype(self.grid.cell_size),
                shape.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(keys.data_ptr()),
                ctypes.c_void_p(oob.data_ptr()), self.stream)
        self._native.check(rc, "cell_keys")
        return keys, oob

    # -- halo plan ----------------------------------------------------------------

    def attach(self, comm):
        """On NCCL runs the library gets its own communicator over the same
        ranks and enqueues every sub-step's halo refreshes itself."""
        if comm.gloo:
            return
        L = self.L
        uid = ctypes.create_string_buffer(int(L.sph_comm_id_bytes()))
        if comm.rank == 0:
            self._native.check(L.sph_comm_unique_id(uid), "comm_unique_id")
        obj = [uid.raw if comm.rank == 0 else None]
        comm.dist.broadcast_object_list(obj, src=0)
        uid = ctypes.create_string_buffer(obj[0], len(obj[0]))
        handle = ctypes.c_void_p()
        self._native.check(L.sph_comm_init(uid, comm.size, comm.rank, ctypes.byref(handle)),
                           "comm_init")
        self.comm_handle = handle
        self.native_loop = True

    def set_halo(self, sel):
        """Device halo plan from the orchestrator's row selections:
        sel[name] = (send rows {q}, ghost rows {q}), name in (fluid, wall)."""
        torch = _torch()
        P = self._native.SphHaloPlan()
        peers = sorted(set(sel["fluid"][0]) | set(sel["fluid"][1]) |
                       set(sel["wall"][0]) | set(sel["wall"][1]))
        if len(peers) > P.MAX_PEERS:
            raise ValueError(f"{len(peers)} halo peers; at most {P.MAX_PEERS}")
        P.npeers = len(peers)
        for k, q in enumerate(peers):
            P.peer[k] = q
        keep = []
        most = 1
        empty = torch.zeros(0, dtype=torch.int64, device=self.device)
        for c, name in enumerate(("fluid", "wall")):
            send, recv = sel[name]
            for side, rows_of, offs in ((0, send, P.send_off), (1, recv, P.recv_off)):
                parts = [rows_of.get(q, empty) for q in peers]
                off = 0
                for k, r in enumerate(parts):
                    offs[c][k] = off
                    off += int(r.numel())
                offs[c][len(peers)] = off
                most = max(most, off)
                rows = torch.cat(parts) if parts else empty
                phys = self.phys_of_row[rows] if rows.numel() else \
                    torch.zeros(1, dtype=torch.int32, device=self.device)
                keep.append(phys)
                if side == 0:
                    P.send_phys[c] = phys.data_ptr()
                else:
                    P.recv_phys[c] = phys.data_ptr()
        w = 9   # widest record (XV)
        self._send_buf = torch.empty(most * w, dtype=self.halo_dtype, device=self.device)
        self._recv_buf = torch.empty(most * w, dtype=self.halo_dtype, device=self.device)
        P.send_buf = self._send_buf.data_ptr()
        P.recv_buf = self._recv_buf.data_ptr()
        self._plan_keep = keep
        self._peers = peers
        self.plan = P

    def _plan_call(self, name, kind, cls):
        rc = getattr(self.L, name)(ctypes.byref(self.E), ctypes.byref(self.plan),
                                   ctypes.c_int32(kind), ctypes.c_int32(cls), self.stream)
        self._native.check(rc, name)

    def halo_pack(self, kind, which):
        """Pack every record of a class; {peer: (n, width) view of the send
        buffer} for a host-side transport."""
        cls = 0 if which == "fluid" else 1
        self._plan_call("sph_halo_pack", kind, cls)
        w = self.halo_width(kind)
        out = {}
        for k, q in enumerate(self._peers):
            a, b = self.plan.send_off[cls][k], self.plan.send_off[cls][k + 1]
            if b > a:
                out[q] = self._send_buf[a * w: b * w].view(b - a, w)
        return out

    def halo_unpack(self, kind, which, got):
        cls = 0 if which == "fluid" else 1
        w = self.halo_width(kind)
        for k, q in enumerate(self._peers):
            a, b = self.plan.recv_off[cls][k], self.plan.recv_off[cls][k + 1]
            if b > a:
                self._recv_buf[a * w: b * w].copy_(got[q].reshape(-1))
        self._plan_call("sph_halo_unpack", kind, cls)

    def substeps(self, half, full, nsub):
        rc = self.L.sph_engine_substeps_slab(ctypes.byref(self.E), self.comm_handle,
                                             ctypes.byref(self.plan), ctypes.c_double(float(half)),
                                             ctypes.c_double(float(full)), ctypes.c_int32(nsub),
                                             self.stream)
        self._native.check(rc, "engine_substeps_slab")

    # -- device row bookkeeping (csrc/slab.cu) -----------------------------------

    device_rows = True

    @property
    def record_words(self):
        return int(self.L.sph_slab_record_words(self.dim, int(self.f64)))

    def _rows(self, fields):
        R = self._native.SphRows()
        for k, f in enumerate(FIELDS):
            R.f[k] = fields[f].data_ptr()
        return R

    def empty_rows(self, n):
        torch = _torch()
        tdt, d = self.halo_dtype, self.dim
        out = {}
        for f in FIELDS:
            if f in ("x", "v", "dvdt"):
                out[f] = torch.empty((n, d), dtype=tdt, device=self.device)
            elif f in INDEX_FIELDS:
                out[f] = torch.empty((n,), dtype=torch.int32, device=self.device)
            else:
                out[f] = torch.empty((n,), dtype=tdt, device=self.device)
        return out

    def classify(self, fields, layout, rank, peers):
        torch = _torch()
        n = int(fields["id"].shape[0])
        G = self._native.SphSlabGeom()
        G.nplanes = int(self.grid.shape[0])
        origin = self.grid.origin.astype(self.np_dtype)
        for k in range(3):
            G.origin[k] = float(origin[k]) if k < self.dim else 0.0
            G.shape[k] = int(self.grid.shape[k]) if k < self.dim else 1
        G.cell_size = float(self.np_dtype(self.grid.cell_size))
        G.nranks, G.rank = layout.nranks, rank
        G.periodic, G.halo = int(layout.periodic), HALO_PLANES
        for k, c in enumerate(layout.cuts):
            G.cuts[k] = int(c)
        G.npeers = len(peers)
        for k, q in enumerate(peers):
            G.peer[k] = q
        P = len(peers)
        lists = torch.empty((3 * P + 1, max(n, 1)), dtype=torch.int32, device=self.device)
        counts = torch.empty(3 * P + 3, dtype=torch.int32, device=self.device)
        rc = self.L.sph_slab_classify(ctypes.byref(G), ctypes.c_void_p(fields["x"].data_ptr()),
                                      ctypes.c_void_p(fields["wall"].data_ptr()), n, self.dim,
                                      int(self.f64), ctypes.c_void_p(lists.data_ptr()),
                                      ctypes.c_void_p(counts.data_ptr()), self.stream)
        self._native.check(rc, "slab_classify")
        return lists, counts.cpu().tolist()

    def pack_rows(self, fields, rows, n, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty((n, self.record_words), dtype=torch.int32, device=self.device)
        if n:
            R = self._rows(fields)
            rc = self.L.sph_slab_pack(ctypes.byref(R), self.dim, int(self.f64),
                                      ctypes.c_void_p(rows.data_ptr()), n,
                                      ctypes.c_void_p(out.data_ptr()), self.stream)
            self._native.check(rc, "slab_pack")
        return out

    def unpack_rows(self, records, fields, off):
        n = int(records.shape[0])
        if n:
            R = self._rows(fields)
            rec = records.contiguous()
            rc = self.L.sph_slab_unpack(ctypes.c_void_p(rec.data_ptr()), n, ctypes.byref(R),
                                        self.dim, int(self.f64), off, self.stream)
            self._native.check(rc, "slab_unpack")

    def gather_rows(self, src, rows, n, dst, off):
        if n:
            Ri, Ro = self._rows(src), self._rows(dst)
            rc = self.L.sph_slab_gather(ctypes.byref(Ri), ctypes.c_void_p(rows.data_ptr()), n,
                                        ctypes.byref(Ro), self.dim, int(self.f64), off,
                                        self.stream)
            self._native.check(rc, "slab_gather")

    def copy_rows(self, src, dst, n):
        for f in FIELDS:
            dst[f][:n].copy_(src[f][:n])

    # -- backend protocol ---------------------------------------------------------

    def load(self, local, n_owned, grid, count_oob=True):
        torch = _torch()
        n = int(local["id"].shape[0])
        wall = local["wall"]
        nf = int((wall == 0).sum())
        self._ensure(n, nf, n - nf)
        if self.id_range:   # global ids; ownership flags by id
            lid = local["id"]
            self.gid_of_lid = None
        else:               # local id = rank of the global id (a 32-bit key sort)
            gid_sorted, order = torch.sort(local["id"])
            lid = torch.empty(n, dtype=torch.int32, device=self.device)
            lid[order] = torch.arange(n, dtype=torch.int32, device=self.device)
            self.gid_of_lid = gid_sorted
        self.n, self.n_own = n, n_owned
        owned = self.T["owned_id"]
        li = lid.to(torch.int64)
        owned[li[n_owned:]] = 0
        owned[li[:n_owned]] = 1
        if n:
            args = [local[f].contiguous() for f in ("x", "v", "rho", "p", "m", "Vol",
                                                    "drho", "dvdt", "rho_scratch")]
            args += [lid, wall.contiguous(), local["nnb"].contiguous(),
                     local["oflow"].contiguous()]
            self._call("sph_engine_push", *[ctypes.c_void_p(a.data_ptr()) for a in args])
            # physical index of every local row (push records refpos = row)
            ref = self.T["refpos"][:n].to(torch.int64)
            self.phys_of_row = torch.empty(n, dtype=torch.int32, device=self.device)
            self.phys_of_row[ref] = torch.arange(n, dtype=torch.int32, device=self.device)
            del args
        self._phys = {}
        self._call("sph_engine_stats", ctypes.c_int32(self._native.STATS_RESET))
        oob = 0
        if n_owned and count_oob:
            _, o = self._keys(local["x"][:n_owned])
            oob = int(o.item())
        return oob

    def prepare(self, step):
        """Lists for the step: exact (skin 0) for initialize, else a skin
        sized from (vmax, amax, dt) as in Simulation._choose_skin."""
        skin = 0.0
        if step is not None:
            vmax, amax, dt = step
            cutoff = float(self.E.cutoff)
            est = vmax * dt + amax * dt * dt
            cap = (0.45 if self.dim == 3 else 1.0) * cutoff
            skin = min(self._skin_factor * est + 0.02 * cutoff, cap)
        self._call("sph_engine_build_lists", ctypes.c_double(skin))

    @property
    def global_stats(self):
        """The statistics are reduced over the ranks on the device (NCCL)."""
        return self.comm_handle is not None

    def _reduce_stats(self, flags):
        if self.comm_handle is not None:
            rc = self.L.sph_stats_allreduce(ctypes.byref(self.E), self.comm_handle,
                                            ctypes.c_int32(flags), self.stream)
            self._native.check(rc, "stats_allreduce")

    def norms(self):
        self._call("sph_engine_stats", ctypes.c_int32(self._native.STATS_NORMS))
        self._reduce_stats(1)
        s = self._stats()
        from .physics import _bits_to_double
        return [_bits_to_double(s.vmax_bits), _bits_to_double(s.amax_bits)]

    def _phase(self, phase, half=0.0, full=0.0):
        self._call("sph_engine_phase", ctypes.c_int32(phase), ctypes.c_double(float(half)),
                   ctypes.c_double(float(full)))

    def shepard(self):
        self._call("sph_engine_shepard")

    def kick_drift(self, half, full):
        self._phase(self._native.PHASE_KICK_DRIFT, half, full)

    def continuity_du(self, full):
        self._phase(self._native.PHASE_CONTINUITY, 0.0, full)

    def wall_pressure(self, initial=False):
        self._phase(self._native.PHASE_INIT_WALL if initial else self._native.PHASE_WALL)

    def momentum_kick(self, half, next_full=None):
        """MOMENTUM (+ KICK); with next_full also the next sub-step's KICK +
        DRIFT of owned fluid (its kick_drift call is then a no-op)."""
        if half is None:
            self._phase(self._native.PHASE_INIT_MOMENTUM)
        elif next_full is not None:
            self._phase(self._native.PHASE_MOMENTUM_NEXT, half, next_full)
        else:
            self._phase(self._native.PHASE_MOMENTUM, half, 0.0)

    def halo_width(self, kind):
        return int(self.L.sph_engine_halo_width(kind))

    def _phys_of(self, rows):
        # the orchestrator's row selections live for the whole step
        key = id(rows)
        hit = self._phys.get(key)
        if hit is None or hit[0] is not rows:
            hit = (rows, self.phys_of_row[rows])
            self._phys[key] = hit
        return hit[1]

    def pack(self, kind, rows):
        torch = _torch()
        k = int(rows.numel())
        out = torch.empty((k, self.halo_width(kind)), dtype=self.halo_dtype, device=self.device)
        if k:
            phys = self._phys_of(rows)
            self._call("sph_engine_pack", ctypes.c_int32(kind), ctypes.c_void_p(phys.data_ptr()),
                       k, ctypes.c_void_p(out.data_ptr()))
        return out

    def unpack(self, kind, rows, buf):
        k = int(rows.numel())
        if k:
            phys = self._phys_of(rows)
            buf = buf.contiguous()
            self._call("sph_engine_unpack", ctypes.c_int32(kind),
                       ctypes.c_void_p(phys.data_ptr()), k, ctypes.c_void_p(buf.data_ptr()))

    def counters(self):
        frac = None
        if self.comm_handle is not None:   # this rank's refreshes drive its skin
            frac = int(self._stats().ndisp) / max(1, self.n)
        self._reduce_stats(2)
        s = self._stats()
        self._call("sph_engine_stats", ctypes.c_int32(self._native.STATS_RESET))
        if frac is None:
            frac = int(s.ndisp) / max(1, self.n)
        if frac > 2e-2:
            self._skin_factor = min(self._skin_factor * 1.5, 16.0)
        return int(s.interactions), int(s.overflow)

    def stability(self):
        if self.n_own == 0 and self.comm_handle is None:
            return np.inf, 0.0
        self._call("sph_engine_stats", ctypes.c_int32(self._native.STATS_NORMS))
        self._reduce_stats(4)
        s = self._stats()
        from .physics import _key_to_double
        rho_min = math.nan if s.nan_flags & 1 else _key_to_double(s.rho_min_key)
        v2 = math.nan if s.nan_flags & 2 else _key_to_double(s.v2max_key)
        return rho_min, v2

    def export_owned(self):
        """Owned particles (rows [0, n_own) of the last load) in registry
        layout with global ids."""
        torch = _torch()
        n, d = self.n, self.dim
        tdt = self.halo_dtype
        out = {}
        for f in FIELDS:
            if f in ("x", "v", "dvdt"):
                out[f] = torch.empty((n, d), dtype=tdt, device=self.device)
            elif f in INDEX_FIELDS:
                out[f] = torch.empty((n,), dtype=torch.int32, device=self.device)
            else:
                out[f] = torch.empty((n,), dtype=tdt, device=self.device)
        if n:
            order = ("x", "v", "rho", "p", "m", "Vol", "drho", "dvdt", "rho_scratch",
                     "id", "wall", "nnb", "oflow")
            self._call("sph_engine_pull", *[ctypes.c_void_p(out[f].data_ptr()) for f in order])
        own = {f: out[f][: self.n_own] for f in FIELDS}
        if self.gid_of_lid is not None:
            own["id"] = self.gid_of_lid[own["id"].to(torch.int64)]
        return own

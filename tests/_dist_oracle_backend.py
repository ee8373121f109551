"""CPU oracle composition implementing the DistributedSimulation backend
protocol (test infrastructure).  Every phase runs the oracle's restated
reference bodies (oracle/sph_oracle.c) over the rank's owned + ghost
particles; the decomposition logic under test is the product's
(paper_2603_11868_b200/distributed.py).  Halo records: XV = (x, v) rows,
RP_* = (rho, p) rows."""

import numpy as np
import torch

from oracle import oracle as O
from paper_2603_11868_b200.distributed import (FIELDS, INDEX_FIELDS, XV, as_tensor,
                                               cell_plane)


class OracleBackend:
    def __init__(self, scalars, sing, grid):
        # scalars = force_args tail (cell_size, cutoff, h, alpha_d, c0, rho0,
        # alpha_visc, eps_h2) in the run dtype; sing: rho0, c0, h, g
        self.sc = scalars
        self.sing = sing
        self.grid = grid
        self.f = None
        self.n_own = 0
        self._inter = 0
        self._ovf = 0
        self.halo_dtype = torch.from_numpy(np.zeros(1, type(scalars[0]))).dtype
        # periodic grids: the oracle's box for every kernel-level call
        dt = np.dtype(type(scalars[0]))
        self.box = O.box_arrays(dt, getattr(grid, "period", None), grid.origin, grid.dim)

    def planes(self, x):
        xn = x.numpy()
        return torch.from_numpy(cell_plane(xn[:, 0], self.grid.origin.astype(xn.dtype)[0],
                                           xn.dtype.type(self.grid.cell_size),
                                           int(self.grid.shape[0])))

    def load(self, local, n_owned, grid):
        self.f = {}
        for k in FIELDS:
            a = local[k].numpy()
            self.f[k] = np.array(a.view(np.uint32) if k in INDEX_FIELDS else a,
                                 copy=True, order="C")
        self.n_own = n_owned
        x = self.f["x"]
        dt = x.dtype.type
        self.origin = grid.origin.astype(x.dtype)
        self.shape = grid.shape_array()
        keys, _ = O.compute_keys(x, self.origin, dt(grid.cell_size), self.shape)
        _, oob_own = O.compute_keys(x[:n_owned], self.origin, dt(grid.cell_size), self.shape)
        self.offsets, self.pids = O.build_cll(keys, grid.cell_count)
        return oob_own

    def prepare(self, step):
        pass

    def _force(self):
        f = self.f
        return (f["x"], f["v"], f["rho"], f["p"], f["m"], f["wall"], f["id"],
                np.asarray(self.sing["g"], f["x"].dtype), self.offsets, self.pids,
                self.origin, self.shape, f["drho"], f["dvdt"], f["nnb"], f["oflow"],
                *self.sc)

    def _ovf_check(self):
        if self.f["oflow"][: self.n_own].any():
            self._ovf = 1

    def norms(self):
        n = self.n_own
        return [O.vmax(self.f["v"][:n]) if n else 0.0,
                O.vmax(self.f["dvdt"][:n]) if n else 0.0]

    def shepard(self):
        f = self.f
        dt = f["x"].dtype.type
        sc = self.sc
        O.sweep("shepard", (f["x"], f["rho"], f["m"], f["wall"], f["id"], self.offsets,
                            self.pids, self.origin, self.shape, f["rho_scratch"],
                            sc[0], sc[1], sc[2], sc[3]), box=self.box)
        f["rho"][:] = f["rho_scratch"]
        O.integrate("density_update", (f["rho"], f["p"], f["drho"], f["wall"], dt(0),
                                       dt(self.sing["c0"]), dt(self.sing["rho0"])), box=self.box)

    def kick_drift(self, half, full):
        f = self.f
        O.integrate("kick", (f["v"], f["dvdt"], f["wall"], half), box=self.box)
        O.integrate("drift", (f["x"], f["v"], f["wall"], full), box=self.box)

    def continuity_du(self, full):
        f = self.f
        dt = f["x"].dtype.type
        O.sweep("continuity", self._force(), box=self.box)
        self._ovf_check()
        O.integrate("density_update", (f["rho"], f["p"], f["drho"], f["wall"], full,
                                       dt(self.sing["c0"]), dt(self.sing["rho0"])), box=self.box)

    def wall_pressure(self, initial=False):
        f = self.f
        O.sweep("wall_pressure", self._force(), box=self.box)
        self._ovf_check()
        n = self.n_own
        w = f["wall"][:n] != 0
        self._inter += int(f["nnb"][:n][w].sum())

    def momentum_kick(self, half, next_full=None):
        # next_full: the engine may fuse the next kick + drift; the oracle
        # composition runs them in the next kick_drift call instead
        f = self.f
        O.sweep("momentum", self._force(), box=self.box)
        self._ovf_check()
        n = self.n_own
        fl = f["wall"][:n] == 0
        s = int(f["nnb"][:n][fl].sum())
        self._inter += s if half is None else 2 * s
        if half is not None:
            O.integrate("kick", (f["v"], f["dvdt"], f["wall"], half), box=self.box)

    def halo_width(self, kind):
        return 2 * self.f["x"].shape[1] if kind == XV else 2

    def pack(self, kind, rows):
        r = rows.numpy()
        f = self.f
        if kind == XV:
            a = np.concatenate([f["x"][r], f["v"][r]], axis=1)
        else:
            a = np.stack([f["rho"][r], f["p"][r]], axis=1)
        return torch.from_numpy(np.ascontiguousarray(a))

    def unpack(self, kind, rows, buf):
        r = rows.numpy()
        b = buf.numpy()
        f = self.f
        if kind == XV:
            d = f["x"].shape[1]
            f["x"][r] = b[:, :d]
            f["v"][r] = b[:, d:]
        else:
            f["rho"][r] = b[:, 0]
            f["p"][r] = b[:, 1]

    def counters(self):
        out = (self._inter, self._ovf)
        self._inter, self._ovf = 0, 0
        return out

    def stability(self):
        n = self.n_own
        if n == 0:
            return np.inf, 0.0
        v = self.f["v"][:n]
        return float(self.f["rho"][:n].min()), float((v * v).sum(axis=1).max())

    def export_owned(self):
        return {k: as_tensor(self.f[k][: self.n_own].copy(), "cpu") for k in FIELDS}

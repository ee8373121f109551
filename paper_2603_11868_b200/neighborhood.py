"""Uniform grid, cell linked list and neighbour search on the device.

Mirror of ``minisph/neighborhood.py``.  ``build_cell_linked_list`` runs the
CUDA key + radix-sort + offsets path (csrc/cll.cu, csrc/sort.cu) and returns
the reference's counting-sort representation: ``offsets`` (exclusive prefix
per cell) and ``particle_ids`` == argsort(keys, kind="stable").  Neighbour
visits come from the device list builder (csrc/nlist.cuh) in ascending
original-id order (neighborhood.py:10-15).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import Staging, device_of, is_tensor, ptr, stream_ptr, workspace
from .execution import ExecutionPolicy

NEIGHBOR_CAPACITY = _native.NEIGHBOR_CAPACITY   # neighborhood.py:30


class NeighborOverflowError(RuntimeError):
    """neighborhood.py:33-34"""


@dataclass(frozen=True)
class UniformGrid:
    """Axis-aligned uniform grid, half-open lower-inclusive cells
    (neighborhood.py:37-63)."""
    origin: np.ndarray
    cell_size: float
    shape: tuple
    # periodic box (not in the reference): per-axis period,
    # 0 = bounded.  None: the reference's bounded grid.
    period: tuple = None

    @property
    def dim(self):
        return len(self.shape)

    @property
    def cell_count(self):
        return int(np.prod(self.shape))

    @staticmethod
    def from_bounds(lower, upper, cell_size):
        lower = np.asarray(lower, dtype=np.float64)
        upper = np.asarray(upper, dtype=np.float64)
        counts = tuple(int(math.ceil((hi - lo) / cell_size)) + 2
                       for lo, hi in zip(lower, upper))
        return UniformGrid(lower - cell_size, float(cell_size), counts)

    def shape_array(self):
        return np.asarray(self.shape, dtype=np.int64)


class CellLinkedList:
    """neighborhood.py:66-73"""
    __slots__ = ("grid", "offsets", "particle_ids", "out_of_bounds")

    def __init__(self, grid, offsets, particle_ids, out_of_bounds=0):
        self.grid = grid
        self.offsets = offsets
        self.particle_ids = particle_ids
        self.out_of_bounds = out_of_bounds


def cell_index_of(grid, position, diagnostics=None):
    """Row-major cell index of one position (host helper, neighborhood.py:87-102)."""
    lin = 0
    clamped = 0
    for k in range(grid.dim):
        c = int(math.floor((position[k] - grid.origin[k]) / grid.cell_size))
        if c < 0:
            c, clamped = 0, 1
        elif c >= grid.shape[k]:
            c, clamped = grid.shape[k] - 1, 1
        lin = lin * grid.shape[k] + c
    if clamped and diagnostics is not None:
        diagnostics[0] += 1
    return lin


def _grid_scalars(grid, dtype):
    dt = np.dtype(dtype).type
    origin = np.zeros(3, dtype=dtype)
    origin[:grid.dim] = grid.origin.astype(dtype)
    shape = np.ones(3, dtype=np.int64)
    shape[:grid.dim] = grid.shape
    return origin, dt(grid.cell_size), shape


def compute_cell_keys(positions, grid, policy=None):
    """Per-particle linear cell keys and the clamp count (neighborhood.py:137-146)."""
    policy = policy or ExecutionPolicy.cuda()
    pos = positions
    n = pos.shape[0]
    if n == 0:
        return np.empty(0, np.int64), 0
    dtype = np.dtype(str(pos.dtype).replace("torch.", ""))
    lib = _native.lib()
    dev = device_of(policy)
    torch = __import__("torch")
    with Staging(dev) as st:
        x = st.to_dev(pos)
        keys = st.empty((n,), torch.int64)
        oob = st.empty((1,), torch.int32)
        oob.zero_()
        origin, cs, shape = _grid_scalars(grid, dtype)
        fn = getattr(lib, f"sph_cell_keys_{_native.sfx(dtype)}")
        rc = fn(ptr(x), n, grid.dim, origin.ctypes.data_as(ctypes.c_void_p), cs,
                shape.ctypes.data_as(ctypes.c_void_p), ptr(keys), ptr(oob),
                stream_ptr(dev))
        _native.check(rc, "compute_cell_keys")
        out = keys.cpu().numpy()
        count = int(oob.cpu().item())
    return out, count


def build_cell_linked_list(policy, positions, grid):
    """Stable counting-sort CLL (neighborhood.py:149-173) on the device.

    Host (numpy) positions give numpy offsets / particle_ids (int64); CUDA
    tensor positions keep the result on the device.
    """
    n = positions.shape[0]
    ncells = grid.cell_count
    on_device = is_tensor(positions)
    if n == 0:
        z = np.zeros(ncells + 1, np.int64)
        return CellLinkedList(grid, z, np.zeros(0, np.int64))
    torch = __import__("torch")
    dtype = np.dtype(str(positions.dtype).replace("torch.", ""))
    lib = _native.lib()
    dev = positions.device if on_device else device_of(policy)
    with Staging(dev) as st:
        x = st.to_dev(positions)
        offsets = torch.empty(ncells + 1, dtype=torch.int64, device=dev)
        pids = torch.empty(n, dtype=torch.int64, device=dev)
        oob = st.empty((1,), torch.int32)
        oob.zero_()
        ws_bytes = lib.sph_cll_workspace_bytes(n, ncells)
        ws = workspace(dev, ws_bytes)
        origin, cs, shape = _grid_scalars(grid, dtype)
        fn = getattr(lib, f"sph_cll_build_{_native.sfx(dtype)}")
        rc = fn(ptr(x), n, grid.dim, origin.ctypes.data_as(ctypes.c_void_p), cs,
                shape.ctypes.data_as(ctypes.c_void_p), ptr(offsets), ptr(pids),
                ptr(oob), ptr(ws), ws_bytes, stream_ptr(dev))
        _native.check(rc, "build_cell_linked_list")
        count = int(oob.cpu().item())
        if not on_device:
            offsets = offsets.cpu().numpy()
            pids = pids.cpu().numpy()
    return CellLinkedList(grid, offsets, pids, count)


def neighbor_lists(policy, positions, ids, cll, cutoff, first=0, count=None):
    """Ordered neighbour lists of particles first..first+count-1.

    Returns (counts int32[count], lists int32[count, 256]); counts are -1 on
    overflow.  Lists hold physical indices j in ascending id order.
    """
    n = positions.shape[0]
    if count is None:
        count = n - first
    torch = __import__("torch")
    dtype = np.dtype(str(positions.dtype).replace("torch.", ""))
    lib = _native.lib()
    dev = positions.device if is_tensor(positions) else device_of(policy)
    grid = cll.grid
    S = _native.sweep_struct(dtype)
    a = S()
    with Staging(dev) as st:
        x = st.to_dev(positions)
        idt = st.to_dev(np.asarray(ids, np.uint32) if not is_tensor(ids) else ids)
        off = st.to_dev(cll.offsets)
        pid = st.to_dev(cll.particle_ids)
        tiles = (count + 31) // 32
        lists = st.empty((max(tiles, 1), NEIGHBOR_CAPACITY, 32), torch.int32)
        cnts = st.empty((max(count, 1),), torch.int32)
        a.x = ptr(x).value
        a.ids = ptr(idt).value
        a.offsets = ptr(off).value
        a.pids = ptr(pid).value
        origin, cs, shape = _grid_scalars(grid, dtype)
        for k in range(3):
            a.origin[k] = origin[k]
            a.shape[k] = shape[k]
        a.cell_size = cs
        a.cutoff = np.dtype(dtype).type(cutoff)
        a.n = n
        a.dim = grid.dim
        fn = getattr(lib, f"sph_neighbors_{_native.sfx(dtype)}")
        rc = fn(ctypes.byref(a), first, count, ptr(lists), ptr(cnts), stream_ptr(dev))
        _native.check(rc, "neighbor_lists")
        c = cnts.cpu().numpy()[:count]
        ell = lists.cpu().numpy()
    # quad tile-ELL [tile][t/4][lane][t%4] -> rows [particle][t]
    tiles_ = ell.shape[0]
    rows = (ell.reshape(tiles_, NEIGHBOR_CAPACITY // 4, 32, 4).transpose(0, 2, 1, 3)
            .reshape(-1, NEIGHBOR_CAPACITY)[:count])
    return c, rows


def collect_neighbors(i, pos, ids, offsets, particle_ids, origin, cell_size,
                      shape, cutoff, buf):
    """neighborhood.py:176-227 signature: fill ``buf`` with packed
    (id << 32 | j) in ascending id order; returns the count or -1."""
    grid = UniformGrid(np.asarray(origin, np.float64), float(cell_size),
                       tuple(int(s) for s in shape))
    cll = CellLinkedList(grid, offsets, particle_ids)
    c, rows = neighbor_lists(ExecutionPolicy.cuda(), pos, ids, cll, cutoff, i, 1)
    cnt = int(c[0])
    if cnt < 0:
        return -1
    js = rows[0, :cnt].astype(np.int64)
    idv = np.asarray(ids)
    buf[:cnt] = (idv[js].astype(np.int64) << 32) | js
    return cnt


def for_each_neighbor(i, positions, cll, cutoff, visit, ids=None):
    """Invoke visit(j, r_ij, unit_ij) for every j != i within the cutoff in
    ascending original-id order (neighborhood.py:230-251)."""
    n = positions.shape[0]
    if ids is None:
        ids = np.arange(n, dtype=np.uint32)
    c, rows = neighbor_lists(ExecutionPolicy.cuda(), positions, ids, cll,
                             cutoff, i, 1)
    cnt = int(c[0])
    if cnt < 0:
        raise NeighborOverflowError(
            f"more than {NEIGHBOR_CAPACITY} neighbors for particle {i}")
    pos = positions.cpu().numpy() if is_tensor(positions) else positions
    for t in range(cnt):
        j = int(rows[0, t])
        diff = pos[i] - pos[j]
        r = float(np.sqrt(np.dot(diff, diff)))
        visit(j, r, diff / r)


def brute_force_neighbors(i, positions, cutoff):
    """Exact O(N) set {j != i : |x_i - x_j| < cutoff} (neighborhood.py:254-260);
    a host-side test oracle, as in the reference."""
    diff = positions - positions[i]
    r2 = np.einsum("ij,ij->i", diff, diff)
    mask = (r2 < cutoff * cutoff) & (r2 > 0.0)
    mask[i] = False
    return set(np.nonzero(mask)[0].tolist())

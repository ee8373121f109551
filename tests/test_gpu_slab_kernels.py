"""The slab bookkeeping kernels (csrc/slab.cu) against a numpy restatement:
classification of rows into per-peer mover / fluid-halo / wall-halo lists,
the kept list and the clamp count (the same binning and halo rules as
distributed.SlabLayout / cell_plane, bounded and periodic), and the record
pack / unpack / gather round trips of every registry field."""

import numpy as np
import pytest

from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.distributed import (FIELDS, INDEX_FIELDS, EngineBackend,
                                               SlabLayout, cell_plane)
from paper_2603_11868_b200.physics import force_scalars

pytestmark = pytest.mark.gpu


def _backend(periodic):
    if periodic:
        cfg = cases.taylor_green_config(3, 16, precision="f32")
    else:
        cfg = cases.kleefsman_config(dp=0.08, precision="f32")
    reg, grid = cases.build_case(cfg)
    sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
    return reg, grid, EngineBackend(force_scalars(reg, grid), sing, grid, "cuda:0")


def _rows(reg, device):
    from paper_2603_11868_b200.distributed import as_tensor
    return {f: as_tensor(reg.raw_view(f), device) for f in FIELDS}


def _clamped(x, grid):
    """Rows whose cell key clamps on some axis (neighborhood.py:79-84)."""
    out = np.zeros(len(x), bool)
    for k in range(grid.dim):
        t = (x[:, k] - np.float32(grid.origin[k])) / np.float32(grid.cell_size)
        f = np.floor(t)
        out |= ~(f >= 0) | (f >= grid.shape[k])
    return out


@pytest.mark.parametrize("periodic", [False, True])
def test_classify_matches_numpy(periodic):
    import torch
    reg, grid, be = _backend(periodic)
    rng = np.random.default_rng(3)
    fields = _rows(reg, be.device)
    n = reg.particle_count
    # jitter positions (some outside the grid) so every class is populated
    x = reg.raw_view("x").copy()
    x += rng.normal(0, 2 * grid.cell_size, x.shape).astype(np.float32)
    fields["x"] = torch.from_numpy(x).to(be.device)
    nplanes = int(grid.shape[0])
    W = 4
    layout = SlabLayout.even(nplanes, W)
    if periodic:
        layout = SlabLayout(layout.cuts, nplanes, True)
    planes = cell_plane(x[:, 0], np.float32(grid.origin[0]), np.float32(grid.cell_size), nplanes)
    owner = layout.owner(planes)
    wall = reg.raw_view("wall") != 0
    for rank in range(W):
        peers = [q for q in range(W) if q != rank]
        lists, cnt = be.classify(fields, layout, rank, peers)
        P = len(peers)
        lists = lists.cpu().numpy()
        keep = owner == rank
        for k, q in enumerate(peers):
            mv = np.sort(lists[3 * k][:cnt[3 * k]])
            assert np.array_equal(mv, np.nonzero(owner == q)[0]), (rank, q)
            halo = keep & layout.halo_mask(q, planes)
            hf = np.sort(lists[3 * k + 1][:cnt[3 * k + 1]])
            hw = np.sort(lists[3 * k + 2][:cnt[3 * k + 2]])
            assert np.array_equal(hf, np.nonzero(halo & ~wall)[0]), (rank, q)
            assert np.array_equal(hw, np.nonzero(halo & wall)[0]), (rank, q)
        kept = np.sort(lists[3 * P][:cnt[3 * P]])
        assert np.array_equal(kept, np.nonzero(keep)[0])
        assert cnt[3 * P + 1] == 0                       # every owner is a peer here
        assert cnt[3 * P + 2] == int(_clamped(x, grid).sum())
    # neighbours only: rows owned by a non-neighbour are flagged
    lists, cnt = be.classify(fields, layout, 0, [1])
    far = int(((owner != 0) & (owner != 1)).sum())
    assert (cnt[4] > 0) == (far > 0)


def test_record_round_trips():
    import torch
    reg, grid, be = _backend(False)
    src = _rows(reg, be.device)
    n = reg.particle_count
    rows = torch.randperm(n, device=be.device)[: n // 3].to(torch.int32)
    rec = be.pack_rows(src, rows, int(rows.numel()))
    assert rec.shape == (rows.numel(), be.record_words)
    dst = be.empty_rows(int(rows.numel()) + 5)
    be.unpack_rows(rec, dst, 5)
    got = be.empty_rows(int(rows.numel()))
    be.gather_rows(src, rows, int(rows.numel()), got, 0)
    idx = rows.to(torch.int64)
    for f in FIELDS:
        want = src[f][idx]
        assert torch.equal(dst[f][5:], want), f
        assert torch.equal(got[f], want), f
    assert be.record_words == (3 * 3 + 6) + 4

"""The periodic-box extension of the oracle (the reference
has no periodic boundaries) and the host-side pieces around it, on CPU:
the restated rules themselves (minimum image, wrapped blocks, drift wrap),
the Taylor-Green case builder, the periodic cell grid, and that periodic
state never leaks into the bounded (reference) restatement."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.neighborhood import UniformGrid


def _sim(dim, n, precision="f32", shift=None, **kw):
    reg, grid = cases.build_case(cases.taylor_green_config(dim, n, precision=precision))
    if shift is not None:
        reg.raw_view("v")[:] += np.asarray(shift[:dim], dtype=reg.dtype)
    return reg, grid, O.OracleSim.from_registry(reg, grid, **kw)


@pytest.mark.parametrize("dim,n", [(2, 24), (3, 12)])
def test_periodic_lattice_has_no_boundary(dim, n):
    """On a periodic lattice every particle has the same neighbour count and
    the continuity rate of a uniform field vanishes exactly."""
    reg, grid = cases.build_case(cases.taylor_green_config(dim, n, precision="f64"))
    reg.raw_view("v")[:] = 0.0
    reg.raw_view("p")[:] = 0.0
    reg.raw_view("rho")[:] = reg.singular("rho0")
    sim = O.OracleSim.from_registry(reg, grid)
    sim.initialize()
    nnb = sim.f["nnb"]
    assert (nnb == nnb[0]).all() and nnb[0] > 0
    # uniform pressure-free field: momentum = g = 0 up to pair-sum cancellation
    assert np.abs(sim.f["dvdt"]).max() < 1e-9


def test_periodic_grid_tiles_the_period():
    g = cases.periodic_grid(1.0, 3, 0.0065)
    s, cs = g.shape[0], np.float32(g.cell_size)
    assert s == int(np.floor(1.0 / 0.0065 / (1 + 1e-6)))
    assert float(cs) * s >= 1.0 and (s - 1) * float(cs) + 0.0065 <= 1.0
    assert g.period == (1.0, 1.0, 1.0) and (g.origin == 0).all()
    with pytest.raises(cases.CaseConfigError):
        cases.periodic_grid(1.0, 2, 0.4)


def test_taylor_green_initial_field():
    cfg = cases.taylor_green_config(3, 8, precision="f64")
    reg, grid = cases.build_case(cfg)
    x, v = reg.view("x"), reg.view("v")
    k = 2 * np.pi
    assert reg.particle_count == 512 and (reg.view("wall") == 0).all()
    assert np.allclose(v[:, 0], np.sin(k * x[:, 0]) * np.cos(k * x[:, 1]) * np.cos(k * x[:, 2]))
    assert np.allclose(v[:, 1], -np.cos(k * x[:, 0]) * np.sin(k * x[:, 1]) * np.cos(k * x[:, 2]))
    assert (v[:, 2] == 0).all()
    # divergence-free discrete field: the mean velocity vanishes
    assert np.abs(v.mean(axis=0)).max() < 1e-12
    with pytest.raises(cases.CaseConfigError):
        cases.build_case(cases.taylor_green_config(2, 8, tank=(1.0, 2.0)))


def test_drift_wraps_and_pairs_are_symmetric():
    reg, grid, sim = _sim(2, 20, shift=(5.0, -3.0))
    sim.initialize()
    for _ in range(30):
        sim.advance()
    x = sim.f["x"]
    assert (x >= 0).all() and (x <= 1).all()
    # particles crossed the faces: positions by id moved by about a period
    x0 = reg.raw_view("x")[np.argsort(reg.raw_view("id"))]
    assert (np.abs(sim.by_id("x") - x0) > 0.5).any()
    # minimum image: a pair across the x face is found from both sides
    pos = np.array([[0.001, 0.5], [0.999, 0.5], [0.5, 0.5]], np.float32)
    ids = np.arange(3, dtype=np.uint32)
    g = cases.periodic_grid(1.0, 2, 0.05)
    keys, _ = O.compute_keys(pos, g.origin.astype(np.float32), np.float32(g.cell_size),
                             np.asarray(g.shape))
    off, pids = O.build_cll(keys, g.cell_count)
    box = O.box_arrays(np.float32, g.period, g.origin, 2)
    args = (ids, off, pids, g.origin.astype(np.float32), np.float32(g.cell_size),
            np.asarray(g.shape), np.float32(0.05))
    c0, n0 = O.collect_neighbors(0, pos, *args, box=box)
    c1, n1 = O.collect_neighbors(1, pos, *args, box=box)
    assert (c0, list(n0)) == (1, [1]) and (c1, list(n1)) == (1, [0])
    # the same call without the box is the reference's bounded search
    assert O.collect_neighbors(0, pos, *args)[0] == 0


def test_periodic_state_does_not_leak_into_bounded_oracle():
    """A periodic simulation between two bounded runs leaves the bounded
    restatement bit-identical (the box is installed per call)."""
    reg, grid = cases.build_case(cases.CaseConfig(case="dambreak2d", dp=0.05,
                                                  precision="f32"))
    a = O.OracleSim.from_registry(reg, grid)
    a.initialize()
    a.advance()
    _, _, p = _sim(2, 16)
    p.initialize()
    p.advance()
    b = O.OracleSim.from_registry(reg, grid)
    b.initialize()
    b.advance()
    for f in ("x", "v", "rho", "p", "dvdt"):
        assert a.f[f].tobytes() == b.f[f].tobytes()

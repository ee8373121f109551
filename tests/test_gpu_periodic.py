"""Periodic boxes (beyond the reference): the CUDA
engine (libsphb200_periodic.so) against the oracle's restatement of the same
extension (oracle/sph_oracle_impl.h: minimum-image pair differences, wrapped
3^d blocks, drift wrap), bit for bit on every field, dt, nsub and the
interaction counts.  A uniform drift is added to the Taylor-Green field so
particles cross every periodic face within the window."""

import numpy as np
import pytest

from _util import FIELDS

import paper_2603_11868_b200 as P
from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.physics import Simulation
from oracle.oracle import OracleSim

pytestmark = pytest.mark.gpu
CUDA = P.ExecutionPolicy.cuda()


def _case(dim, n, precision, shift):
    cfg = cases.taylor_green_config(dim, n, precision=precision)
    reg, grid = cases.build_case(cfg)
    v = reg.raw_view("v")
    v += np.asarray(shift[:dim], dtype=v.dtype)
    return reg, grid


@pytest.mark.parametrize("dim,n,precision,steps,sort_every,shepard_every", [
    (3, 24, "f32", 40, 7, 11),
    (2, 48, "f32", 60, 13, 17),
    (3, 16, "f64", 25, 5, 9),
    (2, 20, "f64", 30, 100, 200),
])
def test_periodic_engine_matches_oracle(dim, n, precision, steps, sort_every,
                                        shepard_every):
    reg, grid = _case(dim, n, precision, (3.0, -2.0, 1.5))
    osim = OracleSim.from_registry(reg, grid, sort_every=sort_every,
                                   shepard_every=shepard_every)
    sim = Simulation(reg, grid, CUDA, sort_every=sort_every,
                     shepard_every=shepard_every)
    osim.initialize()
    sim.initialize()
    assert sim.interaction_count == osim.interaction_count
    x0 = reg.view("x")[np.argsort(reg.view("id"), kind="stable")].copy()
    for step in range(steps):
        dt = sim.advance()
        assert dt == osim.advance(), step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
        if step % 10 == 9 or step == steps - 1:
            for f in FIELDS:
                assert reg.view(f).tobytes() == osim.f[f].tobytes(), (step, f)
            x = reg.view("x")
            assert (x >= 0).all() and (x <= 1).all()
    # particles wrapped: some coordinate jumped by about a period
    x1 = osim.f["x"][np.argsort(osim.f["id"], kind="stable")]
    assert (np.abs(x1 - x0) > 0.5).any()


def test_periodic_lattice_is_homogeneous():
    """Every particle of an unperturbed periodic lattice sees the same
    neighbour count (no boundary deficit): the interaction count of the
    initialisation is exactly N x per-particle count."""
    cfg = cases.taylor_green_config(3, 20, precision="f32")
    reg, grid = cases.build_case(cfg)
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    nnb = reg.view("nnb")
    assert (nnb == nnb[0]).all() and nnb[0] > 0


def test_bounded_library_rejects_periodic_engine():
    from paper_2603_11868_b200 import _native
    from paper_2603_11868_b200.physics import engine_alloc, force_scalars, engine_set_counts
    import ctypes
    import torch
    cfg = cases.taylor_green_config(3, 12, precision="f32")
    reg, grid = cases.build_case(cfg)
    E, T = engine_alloc(torch.device("cuda", 0), reg.particle_count, reg.particle_count, 0,
                        3, False, grid, force_scalars(reg, grid), reg.singular("g"))
    engine_set_counts(E, reg.particle_count, reg.particle_count)
    lib = _native.lib(periodic=False)
    rc = lib.sph_engine_build_lists(ctypes.byref(E), 0.0, None)
    assert rc == _native.SPH_ERR_UNSUPPORTED
    assert "periodic" in _native.last_error()


@pytest.mark.parametrize("mode", ["pass", "queue"])
def test_list_refresh_paths_match_oracle(mode):
    """Both sub-step list-upkeep paths (one-pass check + refresh, and the
    queued k_mark + k_fix_build) under heavy refresh traffic: a drifting
    periodic lattice changes cells every few steps."""
    reg, grid = _case(3, 16, "f32", (6.0, -4.0, 3.0))
    osim = OracleSim.from_registry(reg, grid)
    sim = Simulation(reg, grid, CUDA)
    sim.list_refresh = mode
    osim.initialize()
    sim.initialize()
    nfix = 0
    for step in range(25):
        assert sim.advance() == osim.advance(), step
        assert sim.interaction_count == osim.interaction_count, step
        nfix += sim.last_nfix
    for f in FIELDS:
        assert reg.view(f).tobytes() == osim.f[f].tobytes(), f
    assert nfix > 0

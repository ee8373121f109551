"""The device-resident step engine (physics.Simulation) vs the reference.

Whole-step trajectories against the reference's own fixtures (every discrete
variable by id AND in the registry's physical order, dt, nsub, interaction
and clamp counts), and against the CPU oracle on larger cases and on
configurations the fixtures do not cover.
"""

import numpy as np
import pytest

from _util import FIELDS, TRAJ, by_id, case, golden, mismatched, sha

import paper_2603_11868_b200 as P
from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.physics import (Simulation, SimulationUnstableError,
                                           compute_timestep)
from paper_2603_11868_b200.neighborhood import NeighborOverflowError
from oracle import oracle as O

pytestmark = pytest.mark.gpu
CUDA = P.ExecutionPolicy.cuda()


def _engine_fields(reg):
    return {f: reg.view(f) for f in FIELDS}


@pytest.mark.parametrize("tag", sorted(TRAJ))
def test_engine_trajectory_bitwise_vs_reference(tag):
    z = golden(f"traj_{tag}.npz")
    reg, grid = case(tag)
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    assert sim.interaction_count == z["interactions"][0]
    ids = lambda: reg.view("id")
    assert not mismatched(lambda f: by_id(reg.view(f), ids()), z, 0)
    steps = len(z["dt"]) - 1
    check_every = 1 if steps <= 250 else 10
    for step in range(1, steps + 1):
        dt = sim.advance()
        assert dt == z["dt"][step], step
        assert sim.last_nsub == z["nsub"][step], step
        assert sim.interaction_count == z["interactions"][step], step
        assert sim.out_of_bounds == z["out_of_bounds"][step], step
        if step % check_every == 0 or step == steps:
            bad = mismatched(lambda f: by_id(reg.view(f), ids()), z, step,
                             lambda f: reg.view(f))
            assert not bad, (step, bad)
    for s in z["full_steps"]:
        if s == steps:
            for f in FIELDS:
                assert np.array_equal(by_id(reg.view(f), ids()), z[f"s{s}_{f}"]), f


def test_engine_device_resident_run_matches_golden_without_pulls():
    """No host pulls between steps: the device layout (fluid re-sorted every
    step) is never re-pushed, yet every field matches at the end."""
    tag = "dambreak2d_f32"
    z = golden(f"traj_{tag}.npz")
    reg, grid = case(tag)
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    for _ in range(201):
        sim.advance()
    bad = mismatched(lambda f: by_id(reg.view(f), reg.view("id")), z, 201,
                     lambda f: reg.view(f))
    assert not bad


def _oracle_vs_engine(reg, grid, steps, **kw):
    osim = O.OracleSim.from_registry(reg, grid, **kw)
    sim = Simulation(reg, grid, CUDA, **kw)
    osim.initialize()
    sim.initialize()
    assert sim.interaction_count == osim.interaction_count
    for step in range(steps):
        dt_o = osim.advance()
        dt_g = sim.advance()
        assert dt_g == dt_o, step
        assert sim.last_nsub == osim.last_nsub
        assert sim.interaction_count == osim.interaction_count
        assert sim.out_of_bounds == osim.out_of_bounds
    for f in FIELDS:
        assert reg.view(f).tobytes() == osim.f[f].tobytes(), f


def test_engine_vs_oracle_2d_fine():
    cfg = cases.CaseConfig(case="dambreak2d", dp=0.008, precision="f32")
    reg, grid = cases.build_case(cfg)
    _oracle_vs_engine(reg, grid, 6)


def test_engine_vs_oracle_3d_medium():
    cfg = cases.kleefsman_config(dp=0.02, precision="f32")
    reg, grid = cases.build_case(cfg)
    _oracle_vs_engine(reg, grid, 3)


def test_engine_vs_oracle_sort_and_shepard_cadence():
    cfg = cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f32")
    reg, grid = cases.build_case(cfg)
    _oracle_vs_engine(reg, grid, 25, sort_every=3, shepard_every=4)


def test_engine_vs_oracle_hydrostatic_f64_fixed_dt():
    cfg = cases.CaseConfig(case="hydrostatic", tank=(0.5, 0.6), column=(0.5, 0.5),
                           dp=0.02, hydrostatic_init=True, precision="f64")
    reg, grid = cases.build_case(cfg)
    _oracle_vs_engine(reg, grid, 20, fixed_dt=2e-4)


def test_engine_free_cloud_no_walls_and_clamped_particles():
    """A wall-free cloud partly outside the grid (clamped, counted)."""
    from paper_2603_11868_b200.neighborhood import UniformGrid
    from paper_2603_11868_b200.physics import setup_state_variables
    from paper_2603_11868_b200.variables import VariableRegistry
    rng = np.random.default_rng(5)
    n = 3000
    reg = VariableRegistry(n, 2, dtype=np.float32)
    setup_state_variables(reg)
    reg.raw_view("x")[:] = rng.random((n, 2)) * 1.0
    reg.raw_view("v")[:] = rng.normal(0, 0.3, (n, 2))
    reg.raw_view("rho")[:] = 1000.0
    reg.raw_view("m")[:] = 1000.0 * 0.02 ** 2
    for k, val in (("rho0", 1000.0), ("c0", 20.0), ("h", 0.026), ("dp", 0.02),
                   ("alpha_visc", 0.02)):
        reg.register_singular(k, val)
    reg.register_singular("g", np.array([0.0, -9.81]))
    grid = UniformGrid.from_bounds((0.1, 0.1), (0.9, 0.9), 0.052)
    _oracle_vs_engine(reg, grid, 5)


def test_engine_stability_and_overflow_errors():
    from paper_2603_11868_b200.neighborhood import UniformGrid
    from paper_2603_11868_b200.physics import setup_state_variables
    from paper_2603_11868_b200.variables import VariableRegistry
    rng = np.random.default_rng(8)
    n = 300
    reg = VariableRegistry(n, 2, dtype=np.float32)
    setup_state_variables(reg)
    reg.raw_view("x")[:] = 0.5 + rng.random((n, 2)) * 1e-4
    reg.raw_view("rho")[:] = 1000.0
    reg.raw_view("m")[:] = 1.0
    for k, val in (("rho0", 1000.0), ("c0", 20.0), ("h", 0.065), ("dp", 0.05),
                   ("alpha_visc", 0.02)):
        reg.register_singular(k, val)
    reg.register_singular("g", np.array([0.0, 0.0]))
    grid = UniformGrid.from_bounds((0.3, 0.3), (0.7, 0.7), 0.13)
    sim = Simulation(reg, grid, CUDA)
    with pytest.raises(NeighborOverflowError):
        sim.initialize()
    # absurd fixed dt -> instability (tests/test_harness.py:178-185): the
    # engine aborts at the same step, with the same check, as the oracle
    cfg = cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f32")
    reg2, grid2 = cases.build_case(cfg)
    osim = O.OracleSim.from_registry(reg2, grid2, fixed_dt=0.05)
    sim2 = Simulation(reg2, grid2, CUDA, fixed_dt=0.05)
    osim.initialize()
    sim2.initialize()
    o_fail = g_fail = None
    for step in range(20):
        try:
            osim.advance()
        except O.OracleError as exc:
            o_fail = (step, exc.code)
        try:
            sim2.advance()
        except SimulationUnstableError as exc:
            g_fail = (step, 2 if "density" in str(exc) else 3)
        assert (o_fail is None) == (g_fail is None), (o_fail, g_fail)
        if o_fail:
            break
    assert o_fail == g_fail and o_fail is not None


def test_host_modification_between_steps_is_honoured():
    cfg = cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f32")
    reg, grid = cases.build_case(cfg)
    reg_o, _ = cases.build_case(cfg)
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    sim.advance()
    reg.view("v")[:5] += np.float32(0.25)       # in-place host edit
    osim = O.OracleSim.from_registry(reg, grid)
    osim.st.step_count = sim.step_count
    osim.st.time = sim.time
    dt_g = sim.advance()
    dt_o = osim.advance()
    assert dt_g == dt_o
    for f in ("x", "v", "rho", "p", "dvdt", "drho"):
        assert reg.view(f).tobytes() == osim.f[f].tobytes(), f


def test_compute_timestep_across_policies():
    rng = np.random.default_rng(11)
    cfg = cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f64")
    reg, grid = cases.build_case(cfg)
    reg.view("v")[:] = rng.normal(0.0, 1.0, reg.view("v").shape)
    reg.view("dvdt")[:] = rng.normal(0.0, 10.0, reg.view("dvdt").shape)
    vals = {compute_timestep(p, reg, dt_max=1e-3)
            for p in (P.ExecutionPolicy.sequenced(), P.ExecutionPolicy.parallel(4), CUDA)}
    assert len(vals) == 1
    vm = O.vmax(reg.view("v"))
    am = O.vmax(reg.view("dvdt"))
    from paper_2603_11868_b200.physics import timestep_formula
    assert vals.pop() == timestep_formula(vm, am, float(reg.singular("h")),
                                          float(reg.singular("c0")), 1e-3)


def _cloud(n, dim, dtype, seed, wall_frac=0.0, spread=1.0, coincident=0):
    """A random particle cloud registry (+ optional walls and coincident
    pairs) on a grid covering most of it."""
    from paper_2603_11868_b200.neighborhood import UniformGrid
    from paper_2603_11868_b200.physics import setup_state_variables
    from paper_2603_11868_b200.variables import VariableRegistry
    rng = np.random.default_rng(seed)
    reg = VariableRegistry(n, dim, dtype=dtype)
    setup_state_variables(reg)
    x = rng.random((n, dim)) * spread
    if coincident and n > 2 * coincident:
        x[n - coincident:] = x[:coincident]          # exact duplicates
    reg.raw_view("x")[:] = x
    reg.raw_view("v")[:] = rng.normal(0, 0.2, (n, dim))
    reg.raw_view("rho")[:] = 1000.0 + rng.normal(0, 2.0, n)
    reg.raw_view("m")[:] = 1000.0 * 0.02 ** dim
    if wall_frac:
        reg.raw_view("wall")[:] = (rng.random(n) < wall_frac).astype(np.uint32)
    reg.raw_view("id")[:] = rng.permutation(n).astype(np.uint32)
    for k, val in (("rho0", 1000.0), ("c0", 20.0), ("h", 0.026), ("dp", 0.02),
                   ("alpha_visc", 0.02)):
        reg.register_singular(k, val)
    g = np.zeros(dim)
    g[-1] = -9.81
    reg.register_singular("g", g)
    grid = UniformGrid.from_bounds(np.full(dim, 0.05), np.full(dim, 0.95) * spread, 0.052)
    return reg, grid


@pytest.mark.parametrize("dim,dtype", [(2, np.float32), (3, np.float32), (3, np.float64)])
def test_engine_vs_oracle_random_clouds_with_walls_and_duplicates(dim, dtype):
    """Scrambled ids, a quarter walls scattered through the fluid, exactly
    coincident particles (r2 = 0: never neighbours, but inside skin lists)."""
    n = 4000 if dim == 2 else 6000
    reg, grid = _cloud(n, dim, dtype, seed=11 + dim, wall_frac=0.25,
                       spread=1.0 if dim == 2 else 0.5, coincident=50)
    _oracle_vs_engine(reg, grid, 6)


def test_engine_walls_only_and_single_particle():
    """Degenerate sizes: no fluid at all; one fluid particle (no neighbours)."""
    reg, grid = _cloud(500, 2, np.float32, seed=3)
    reg.raw_view("wall")[:] = 1
    _oracle_vs_engine(reg, grid, 3)
    reg, grid = _cloud(1, 2, np.float32, seed=4)
    _oracle_vs_engine(reg, grid, 3)


def test_engine_empty_registry():
    reg, grid = _cloud(0, 2, np.float32, seed=5)
    osim = O.OracleSim.from_registry(reg, grid)
    sim = Simulation(reg, grid, CUDA)
    osim.initialize()
    sim.initialize()
    for _ in range(2):
        assert sim.advance() == osim.advance()
    assert sim.interaction_count == osim.interaction_count == 0


def test_push_checks_ids_and_follows_wall_flag_edits():
    """The registry checks run on the device at push: a non-permutation of
    ids raises ValueError; edited wall flags resize the engine."""
    reg, grid = _cloud(2000, 2, np.float32, seed=21, wall_frac=0.2)
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    sim.advance()
    ids = reg.view("id")
    saved = ids.copy()
    ids[0] = ids[1]
    with pytest.raises(ValueError):
        sim.advance()
    reg.view("id")[:] = saved
    wall = reg.view("wall")
    wall[:60] ^= 1
    osim = O.OracleSim.from_registry(reg, grid)
    osim.st.step_count = sim.step_count
    osim.st.time = sim.time
    for _ in range(3):
        assert sim.advance() == osim.advance()
    for f in FIELDS:
        assert reg.view(f).tobytes() == osim.f[f].tobytes(), f


@pytest.mark.parametrize("kind", ["3d", "2d"])
def test_engine_lists_carried_across_steps_vs_oracle(kind, monkeypatch):
    """Skin lists kept across advective steps (sph_engine_maintain_lists:
    renumbered through the re-sort, leavers dropped, arriving movers merged
    by id) must give the reference's neighbour sets: long epochs with a wide
    skin force many carried steps, movers and refreshes."""
    from paper_2603_11868_b200 import physics
    monkeypatch.setattr(physics, "LIST_EPOCH_STEPS", 8)
    monkeypatch.setattr(physics, "LIST_EPOCH_LIMIT", 0.9)
    monkeypatch.setattr(physics, "LIST_EPOCH_REFRESH", 1.0)   # carry regardless of refreshes
    monkeypatch.setattr(physics, "LIST_EPOCH_MAX", 10)
    monkeypatch.setenv("SPH_LIST_EPOCHS", "always")
    if kind == "3d":
        cfg, steps = cases.kleefsman_config(dp=0.02, precision="f32"), 40
    else:
        cfg, steps = cases.CaseConfig(case="dambreak2d", dp=0.01, precision="f32"), 80
    reg, grid = cases.build_case(cfg)
    osim = O.OracleSim.from_registry(reg, grid)
    sim = Simulation(reg, grid, CUDA)
    osim.initialize()
    sim.initialize()
    modes = []
    for step in range(steps):
        assert sim.advance() == osim.advance(), step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        modes.append(sim.last_list_mode)
    assert modes.count("maintain") >= steps // 3, modes
    for f in FIELDS:
        assert reg.view(f).tobytes() == osim.f[f].tobytes(), f


def test_engine_lists_carried_with_clamped_free_cloud(monkeypatch):
    """Random velocities (many movers per step, particles leaving the grid
    and clamping) through carried lists."""
    from paper_2603_11868_b200 import physics
    from paper_2603_11868_b200.neighborhood import UniformGrid
    from paper_2603_11868_b200.variables import VariableRegistry
    monkeypatch.setattr(physics, "LIST_EPOCH_STEPS", 6)
    monkeypatch.setattr(physics, "LIST_EPOCH_LIMIT", 0.9)
    monkeypatch.setattr(physics, "LIST_EPOCH_REFRESH", 1.0)
    monkeypatch.setattr(physics, "LIST_EPOCH_MAX", 10)
    monkeypatch.setenv("SPH_LIST_EPOCHS", "always")
    rng = np.random.default_rng(11)
    n = 4000
    reg = VariableRegistry(n, 3, dtype=np.float32)
    physics.setup_state_variables(reg)
    reg.raw_view("x")[:] = rng.random((n, 3)) * 0.6
    reg.raw_view("v")[:] = rng.normal(0, 0.05, (n, 3))
    reg.raw_view("rho")[:] = 1000.0
    reg.raw_view("m")[:] = 1000.0 * 0.02 ** 3
    for k, val in (("rho0", 1000.0), ("c0", 20.0), ("h", 0.026), ("dp", 0.02),
                   ("alpha_visc", 0.02)):
        reg.register_singular(k, val)
    reg.register_singular("g", np.array([0.0, 0.0, -9.81]))
    grid = UniformGrid.from_bounds((0.05, 0.05, 0.05), (0.55, 0.55, 0.55), 0.052)
    osim = O.OracleSim.from_registry(reg, grid)
    sim = Simulation(reg, grid, CUDA)
    osim.initialize()
    sim.initialize()
    modes = []
    for step in range(25):
        assert sim.advance() == osim.advance(), step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
        modes.append(sim.last_list_mode)
    assert "maintain" in modes, modes
    for f in FIELDS:
        assert reg.view(f).tobytes() == osim.f[f].tobytes(), f


def test_engine_vs_oracle_3d_f64():
    """precision="f64" (every operation binary64) on
    the 3D Kleefsman case with walls and the obstacle."""
    cfg = cases.kleefsman_config(dp=0.04, precision="f64")
    reg, grid = cases.build_case(cfg)
    _oracle_vs_engine(reg, grid, 8)

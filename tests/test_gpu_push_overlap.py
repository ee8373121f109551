"""The overlapped host push and pull (physics.Simulation._push_overlapped,
_pull_overlapped).

A step that starts from host-authoritative state (the registry was viewed,
and so may have been edited, since the last step) uploads x, id and wall
first, lays the particles out and builds the step's skin lists while the
other ten fields are still in flight, and skips the step's CLL re-sort (the
push's cell order is that CLL).  These tests hold it to the plain push
(sph_engine_push + rebuild + lists sized by this step's dt) bit for bit,
every field every step, plus dt, nsub and the interaction and clamp counts,
and to the CPU oracle on a clamped cloud.  With the registry in pinned
memory and its result viewed after every step, the step also pulls its own
result (x and rho / p / drho during the last momentum sweep), which the
same comparisons cover.
"""

import ctypes

import numpy as np
import pytest

from _util import FIELDS

import paper_2603_11868_b200 as P
from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.physics import Simulation
from oracle import oracle as O

pytestmark = pytest.mark.gpu
CUDA = P.ExecutionPolicy.cuda()


def _clamped_cloud():
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
    return reg, grid


def _pin(reg):
    """Registry storage -> pinned host memory (as bench.py's e2e arm)."""
    import torch
    for name in reg.discrete_names():
        var = reg._discrete[name]
        a = var.data
        t = torch.empty(a.shape, dtype=torch.int32 if a.dtype == np.uint32
                        else torch.from_numpy(a[:0]).dtype, pin_memory=True)
        pinned = t.numpy().view(a.dtype)
        pinned[...] = a
        var.data = pinned
    return reg


CASES = {
    "2d_sort_shepard": (lambda: cases.build_case(
        cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f32")),
        dict(sort_every=3, shepard_every=4), 14),
    "3d": (lambda: cases.build_case(cases.kleefsman_config(dp=0.03, precision="f32")), {}, 4),
    "3d_f64": (lambda: cases.build_case(cases.kleefsman_config(dp=0.04, precision="f64")), {}, 3),
    "clamped_cloud": (_clamped_cloud, {}, 6),
    "taylor_green_periodic": (lambda: cases.build_case(
        cases.taylor_green_config(3, 24, precision="f32")), {}, 4),
}


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("name", sorted(CASES))
def test_overlapped_push_matches_plain_push(name, pinned):
    make, kw, steps = CASES[name]
    reg_a, grid = make()
    reg_b, _ = make()
    if pinned:
        _pin(reg_a)
    a = Simulation(reg_a, grid, CUDA, **kw)
    b = Simulation(reg_b, grid, CUDA, **kw)
    b.push_overlap = False
    b.eager_pull = False
    a.initialize()
    b.initialize()
    for step in range(steps):
        assert a.advance() == b.advance(), step
        assert a.last_push_overlapped == (step > 0), step   # step 0: no dt forecast yet
        # the result of each of the two previous steps was viewed
        assert a.last_pull_overlapped == (pinned and step >= 2), step
        assert not b.last_push_overlapped and not b.last_pull_overlapped
        assert a.last_nsub == b.last_nsub, step
        assert a.interaction_count == b.interaction_count, step
        assert a.out_of_bounds == b.out_of_bounds, step
        # views pull: host-authoritative again, so the next step pushes
        bad = [f for f in FIELDS if reg_a.view(f).tobytes() != reg_b.view(f).tobytes()]
        assert not bad, (step, bad)
    if name == "clamped_cloud":
        assert a.out_of_bounds > 0
    # then no views: after the first step (which still pushes the viewed
    # registry), the device stays authoritative -- nothing is pushed or pulled
    for step in range(3):
        assert a.advance() == b.advance()
        if step:
            assert not a.last_push_overlapped and not a.last_pull_overlapped
    bad = [f for f in FIELDS if reg_a.view(f).tobytes() != reg_b.view(f).tobytes()]
    assert not bad, bad


@pytest.mark.parametrize("pinned", [False, True])
def test_overlapped_push_with_host_edits_vs_oracle(pinned):
    """Edits between steps (velocities, a position out of the grid) reach
    the overlapped push, also after a step that pulled its own result; the
    clamp count follows the oracle's."""
    reg, grid = _clamped_cloud()
    if pinned:
        _pin(reg)
    sim = Simulation(reg, grid, CUDA)
    osim = O.OracleSim.from_registry(reg, grid)
    sim.initialize()
    osim.initialize()
    for step in range(5):
        if step >= 2:   # the same in-place edits on both sides
            for v, x in ((reg.view("v"), reg.view("x")), (osim.f["v"], osim.f["x"])):
                v[step::97] *= np.float32(0.5)
                x[step * 7] = np.float32(-0.25)
        assert sim.advance() == osim.advance(), step
        assert sim.last_push_overlapped == (step > 0), step
        assert sim.last_pull_overlapped == (pinned and step >= 2), step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
        bad = [f for f in FIELDS if reg.view(f).tobytes() != osim.f[f].tobytes()]
        assert not bad, (step, bad)


@pytest.mark.parametrize("bad_id", ["duplicate", "out_of_range"])
def test_overlapped_push_rejects_bad_ids_and_recovers(bad_id):
    """The id check of an overlapped push is read after the step's list
    build was queued: a duplicate or out-of-range id still raises
    ValueError (no device fault), and once the ids are repaired the run goes
    on bit for bit with the oracle."""
    reg, grid = cases.build_case(cases.CaseConfig(case="dambreak2d", dp=0.05,
                                                  precision="f32"))
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    sim.advance()
    ids = reg.view("id")
    saved = ids.copy()
    ids[3] = ids[4] if bad_id == "duplicate" else np.uint32(10 ** 9)
    with pytest.raises(ValueError):
        sim.advance()
    reg.view("id")[:] = saved
    osim = O.OracleSim.from_registry(reg, grid)
    osim.st.step_count = sim.step_count
    osim.st.time = sim.time
    for step in range(3):
        assert sim.advance() == osim.advance(), step
        assert sim.last_push_overlapped   # every step follows a view
        for f in FIELDS:
            assert reg.view(f).tobytes() == osim.f[f].tobytes(), (step, f)


def test_cll_fresh_flag_follows_particle_motion():
    """SphEngine.cll_fresh (list builds on a fresh CLL take each particle's
    cell from the CLL instead of recomputing it): set by a push and by a CLL
    rebuild, cleared by anything that moves particles."""
    from paper_2603_11868_b200 import _native
    reg, grid = cases.build_case(cases.CaseConfig(case="dambreak2d", dp=0.05,
                                                  precision="f32"))
    sim = Simulation(reg, grid, CUDA)
    sim.initialize()
    E = sim._dev["E"]
    assert E.cll_fresh == 1          # push + rebuild, then the initial sweeps move nothing
    sim.advance()
    assert E.cll_fresh == 0          # the step's sub-steps drifted the particles
    sim._rebuild_cll()
    assert E.cll_fresh == 1
    sim._build_lists(0.0)            # a list build moves nothing
    assert E.cll_fresh == 1
    sim._call("sph_engine_phase", ctypes.c_int32(_native.PHASE_KICK_DRIFT),
              ctypes.c_double(1e-6), ctypes.c_double(2e-6))
    assert E.cll_fresh == 0
    reg.view("x")                    # pull, then the next step pushes
    sim.advance()
    assert E.cll_fresh == 0 and sim.last_push_overlapped

"""Bitwise parity at the benchmark configurations (BASELINE.json configs 2-5).

bench.py times the engine on the 2D 1M, 3D 4M and 3D 16M dam breaks, built
on the device (cases.build_case_device).  These tests run exactly that path
(device placement -> Simulation.load_device_state -> initialize -> advance)
next to the CPU oracle (OracleSim, the C restatement of
physics.py:460-552 pinned to the reference's goldens) on the host-built
case, and compare every discrete variable byte for byte after each window,
plus dt, nsub, the cumulative interaction and clamp counts at every step.

The 1M / 4M / 16M sizes exercise engine paths the small goldens cannot:
oversized candidate blocks (k_skin_big), the one-pass vs queued list refresh
choice, the split-filter threshold and multi-wave grids.
Reference: /root/reference/pkg/src/minisph/physics.py:489-552.
"""

import os

import numpy as np
import pytest

import paper_2603_11868_b200 as P
from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.physics import Simulation
from oracle import oracle as O

from _util import FIELDS

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# (config, builder, steps) -- oracle cost on 16 host threads: ~2 s, ~6 s and
# ~40 s per advective step
BENCH_CASES = {
    "2d1m": (lambda: cases.CaseConfig(case="dambreak2d", dp=0.00144, precision="f32"), 3),
    "3d4m": (lambda: cases.kleefsman_config(dp=0.00608, precision="f32"), 3),
    "3d16m": (lambda: cases.kleefsman_config(dp=0.00371, precision="f32"), 1),
}


def _run(name):
    import torch
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    make, steps = BENCH_CASES[name]
    cfg = make()
    reg_h, grid_h = cases.build_case(cfg)
    osim = O.OracleSim.from_registry(reg_h, grid_h)
    del reg_h
    reg, grid, state = cases.build_case_device(cfg, torch.device("cuda", 0))
    assert np.array_equal(grid.shape, grid_h.shape) and \
        np.array_equal(grid.origin, grid_h.origin)
    sim = Simulation(reg, grid, P.ExecutionPolicy.cuda(0))
    sim.load_device_state(state)
    del state
    osim.initialize()
    sim.initialize()
    assert sim.interaction_count == osim.interaction_count
    for step in range(steps):
        dt_o = osim.advance()
        dt_g = sim.advance()
        assert dt_g == dt_o, step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
    bad = [f for f in FIELDS if reg.view(f).tobytes() != osim.f[f].tobytes()]
    assert not bad, bad
    # neighbour counts are exact: the per-particle lists the sweeps used
    assert int(reg.view("nnb").sum()) == int(osim.f["nnb"].sum())


def test_bench_config2_2d1m_bitwise_vs_oracle():
    _run("2d1m")


def test_bench_config3_3d4m_bitwise_vs_oracle():
    _run("3d4m")


def test_bench_config4_3d16m_bitwise_vs_oracle():
    _run("3d16m")


def test_bench_config5_taylor_green_8m_bitwise_vs_oracle():
    """bench.py --config tg8m: the 200^3 periodic Taylor-Green box on one GPU
    (libsphb200_periodic.so, host placement as the bench) against the
    oracle's periodic restatement for two steps (nsub 3)."""
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    cfg = cases.taylor_green_config(3, 200, precision="f32")
    reg, grid = cases.build_case(cfg)
    osim = O.OracleSim.from_registry(reg, grid)
    sim = Simulation(reg, grid, P.ExecutionPolicy.cuda(0))
    osim.initialize()
    sim.initialize()
    assert sim.interaction_count == osim.interaction_count
    for step in range(2):
        assert sim.advance() == osim.advance(), step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
    bad = [f for f in FIELDS if reg.view(f).tobytes() != osim.f[f].tobytes()]
    assert not bad, bad


def test_bench_window_config3_bitwise_vs_oracle():
    """The bench's whole measured window at config 3 -- initialize, W = 5
    warm-up and K = 20 timed steps (nsub 7-8) -- step for step against the
    oracle: dt, nsub, interaction and clamp counts every step, every field
    at the end (~2.5 min of oracle time on 16 threads)."""
    import torch
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    cfg = BENCH_CASES["3d4m"][0]()
    reg_h, grid_h = cases.build_case(cfg)
    osim = O.OracleSim.from_registry(reg_h, grid_h)
    del reg_h
    reg, grid, state = cases.build_case_device(cfg, torch.device("cuda", 0))
    sim = Simulation(reg, grid, P.ExecutionPolicy.cuda(0))
    sim.load_device_state(state)
    del state
    osim.initialize()
    sim.initialize()
    nsubs = []
    for step in range(25):
        assert sim.advance() == osim.advance(), step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
        nsubs.append(sim.last_nsub)
    assert nsubs[5:] == [7] * 9 + [8] * 11   # the bench line's nsub_per_step
    bad = [f for f in FIELDS if reg.view(f).tobytes() != osim.f[f].tobytes()]
    assert not bad, bad


def test_bench_config2_e2e_path_bitwise_vs_oracle():
    """bench.py's e2e arm at config 2: host-built registry in pinned memory,
    every field viewed after every step -- so steps from the second on push
    with the overlapped upload and from the third on pull their own result
    during the last momentum sweep -- step for step against the oracle."""
    import torch
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    cfg = BENCH_CASES["2d1m"][0]()
    reg, grid = cases.build_case(cfg)
    osim = O.OracleSim.from_registry(reg, grid)
    for name in reg.discrete_names():   # pinned registry storage (bench.pinned_like)
        var = reg._discrete[name]
        a = var.data
        t = torch.empty(a.shape, dtype=torch.int32 if a.dtype == np.uint32
                        else torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy().view(a.dtype)[...] = a
        var.data = t.numpy().view(a.dtype)
    sim = Simulation(reg, grid, P.ExecutionPolicy.cuda(0))
    osim.initialize()
    sim.initialize()
    for step in range(5):
        assert sim.advance() == osim.advance(), step
        assert sim.last_push_overlapped == (step > 0), step
        assert sim.last_pull_overlapped == (step > 1), step
        assert sim.last_nsub == osim.last_nsub, step
        assert sim.interaction_count == osim.interaction_count, step
        assert sim.out_of_bounds == osim.out_of_bounds, step
        bad = [f for f in FIELDS if reg.view(f).tobytes() != osim.f[f].tobytes()]
        assert not bad, (step, bad)

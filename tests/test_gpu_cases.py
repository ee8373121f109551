"""Device case placement (csrc/cases.cu) vs the host
builder restating cases.py:129-238 (itself pinned to the reference's initial
states by the trajectory goldens): every registry field bit for bit, and a
simulation started from the device state steps bit-identically to one
started from the host registry."""

import numpy as np
import pytest

from _util import FIELDS

import paper_2603_11868_b200 as P
from paper_2603_11868_b200 import cases
from paper_2603_11868_b200.physics import Simulation

pytestmark = pytest.mark.gpu
CUDA = P.ExecutionPolicy.cuda()


def _cfgs():
    return {
        "dambreak2d_f32": cases.CaseConfig(case="dambreak2d", precision="f32"),
        "dambreak2d_f64_fine": cases.CaseConfig(case="dambreak2d", dp=0.0123,
                                                precision="f64"),
        "offset2d": cases.CaseConfig(case="dambreak2d", dp=0.05, precision="f32",
                                     column_offset=(1.01, 0.3)),
        "hydrostatic_f32": cases.CaseConfig(
            case="hydrostatic", tank=(1.0, 1.2), column=(1.0, 1.0), dp=0.02,
            hydrostatic_init=True, precision="f32"),
        "hydrostatic_f64": cases.CaseConfig(
            case="hydrostatic", tank=(1.0, 1.2), column=(1.0, 1.0), dp=0.031,
            hydrostatic_init=True, precision="f64"),
        "kleefsman_f32": cases.kleefsman_config(dp=0.04, precision="f32"),
        "kleefsman_f32_fine": cases.kleefsman_config(dp=0.0173, precision="f32"),
        "kleefsman_hydro_f64": cases.kleefsman_config(dp=0.05, precision="f64",
                                                      hydrostatic_init=True),
    }


@pytest.mark.parametrize("tag", sorted(_cfgs()))
def test_device_case_equals_host_case(tag):
    cfg = _cfgs()[tag]
    reg, grid = cases.build_case(cfg)
    dreg, dgrid, st = cases.build_case_device(cfg)
    assert dreg.particle_count == reg.particle_count
    assert np.array_equal(dgrid.origin, grid.origin)
    assert np.array_equal(dgrid.shape, grid.shape)
    assert dgrid.cell_size == grid.cell_size
    for f in FIELDS:
        host = reg.raw_view(f)
        dev = st[f].cpu().numpy()
        if host.dtype == np.uint32:
            dev = dev.view(np.uint32)
        assert dev.dtype == host.dtype and dev.shape == host.shape, f
        assert dev.tobytes() == host.tobytes(), f
    for name in ("rho0", "c0", "h", "dp", "alpha_visc"):
        assert dreg.singular(name) == reg.singular(name)
    assert np.array_equal(dreg.singular("g"), reg.singular("g"))


@pytest.mark.parametrize("tag", ["dambreak2d_f32", "kleefsman_f32"])
def test_simulation_from_device_state_matches_host(tag):
    cfg = _cfgs()[tag]
    reg, grid = cases.build_case(cfg)
    dreg, dgrid, st = cases.build_case_device(cfg)
    a = Simulation(reg, grid, CUDA)
    b = Simulation(dreg, dgrid, CUDA)
    b.load_device_state(st)
    del st
    a.initialize()
    b.initialize()
    for _ in range(3):
        assert a.advance() == b.advance()
        assert a.last_nsub == b.last_nsub
    assert a.interaction_count == b.interaction_count
    for f in FIELDS:
        assert reg.view(f).tobytes() == dreg.view(f).tobytes(), f


def test_lattice_modes_edge_cases():
    """Empty boxes, a single point, negative ranges, the tank test on a
    ragged box and the open-box cut, against a numpy restatement."""
    import torch
    dev = torch.device("cuda", 0)
    dp = 0.0371
    for ranges in ([(0, 0), (0, 5)], [(3, 4), (-2, -1)], [(-3, 7), (-3, 11)],
                   [(-2, 5), (-2, 4), (-2, 3)], [(0, 1), (0, 1), (0, 1)]):
        d = len(ranges)
        anchor = np.linspace(-0.3, 0.7, d)
        want = cases._lattice(ranges, dp, anchor)
        got, _ = cases._device_lattice(dev, ranges, dp, anchor)
        assert got.cpu().numpy().tobytes() == np.ascontiguousarray(want).tobytes()
        counts = [max(0, r[1] - 2) for r in ranges]
        pts = cases._lattice(ranges, dp, np.zeros(d))
        if pts.shape[0]:
            idx = np.round(pts / dp - 0.5).astype(np.int64)
            outside = (idx < 0).any(axis=1)
            for k in range(d - 1):
                outside |= idx[:, k] >= counts[k]
            want = pts[outside]
        else:
            want = pts
        got, _ = cases._device_lattice(dev, ranges, dp, np.zeros(d), 1, counts=counts)
        assert got.cpu().numpy().tobytes() == np.ascontiguousarray(want).tobytes()
        lo = anchor + 2.1 * dp
        hi = lo + 3.3 * dp
        pts = cases._lattice(ranges, dp, anchor)
        inside = ((pts > lo) & (pts < hi)).all(axis=1) if pts.shape[0] else np.zeros(0, bool)
        got, _ = cases._device_lattice(dev, ranges, dp, anchor, 2, box=(lo, hi))
        assert got.cpu().numpy().tobytes() == np.ascontiguousarray(pts[~inside]).tobytes()

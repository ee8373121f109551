"""The slab path's NCCL transport on one GPU (csrc/halo.cu): a one-rank NCCL
communicator, records sent to the rank itself through the halo plan, and the
one-call-per-step sub-step loop.  Multi-GPU runs use the same plan, packing
and offsets with real peers; the multi-rank decomposition itself is pinned
by tests/test_gpu_distributed.py."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2603_11868_b200 import ExecutionPolicy, _native, cases
from paper_2603_11868_b200.physics import Simulation

pytestmark = pytest.mark.gpu


def _sim(dp=0.05):
    reg, grid = cases.build_case(cases.CaseConfig(case="dambreak2d", dp=dp, precision="f32"))
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    sim.advance()
    return sim


def _comm1():
    L = _native.lib()
    uid = ctypes.create_string_buffer(int(L.sph_comm_id_bytes()))
    _native.check(L.sph_comm_unique_id(uid), "uid")
    h = ctypes.c_void_p()
    _native.check(L.sph_comm_init(uid, 1, 0, ctypes.byref(h)), "init")
    return h


def test_self_exchange_moves_records_between_particles():
    sim = _sim()
    d = sim._dev
    E, T = d["E"], d["T"]
    L = _native.lib()
    nf = E.nf
    rng = np.random.default_rng(5)
    perm = rng.permutation(nf)
    src = torch.tensor(perm[:40], dtype=torch.int32, device="cuda")
    dst = torch.tensor(perm[40:80], dtype=torch.int32, device="cuda")
    P = _native.SphHaloPlan()
    P.npeers = 1
    P.peer[0] = 0
    for c in range(2):
        P.send_off[c][0] = P.recv_off[c][0] = 0
        P.send_off[c][1] = P.recv_off[c][1] = 40 if c == 0 else 0
        P.send_phys[c] = src.data_ptr()
        P.recv_phys[c] = dst.data_ptr()
    sbuf = torch.zeros(40 * 9, dtype=torch.float32, device="cuda")
    rbuf = torch.zeros(40 * 9, dtype=torch.float32, device="cuda")
    P.send_buf, P.recv_buf = sbuf.data_ptr(), rbuf.data_ptr()
    comm = _comm1()
    pos = T["pos0"] if E.cur_pos == 0 else T["pos1"]
    vel = T["vel0"] if E.cur_v == 0 else T["vel1"]
    before_p = pos[src.long()].clone()
    before_v = vel[src.long()].clone()
    before_d = T["disp"][src.long()].clone()
    rc = L.sph_halo_exchange(ctypes.byref(E), comm, ctypes.byref(P), _native.HALO_XV, 0,
                             d["stream"])
    _native.check(rc, "halo_exchange")
    torch.cuda.synchronize()
    assert torch.equal(pos[dst.long()], before_p)
    assert torch.equal(vel[dst.long()], before_v)
    assert torch.equal(T["disp"][dst.long()], before_d)
    rp_next = T["rp1"] if E.cur_rp == 0 else T["rp0"]
    before_rp = rp_next[src.long()].clone()
    rc = L.sph_halo_exchange(ctypes.byref(E), comm, ctypes.byref(P), _native.HALO_RP_NEXT, 0,
                             d["stream"])
    _native.check(rc, "halo_exchange")
    torch.cuda.synchronize()
    assert torch.equal(rp_next[dst.long()], before_rp)
    rq = T["rq"][dst.long()]
    assert torch.equal(rq[:, 0], before_rp[:, 0])
    _native.check(L.sph_comm_destroy(comm), "destroy")


def test_slab_substep_loop_without_peers_matches_the_engine():
    ref = _sim(0.04)
    for _ in range(4):
        ref.advance()
    L = _native.lib()
    comm = _comm1()
    P = _native.SphHaloPlan()
    P.npeers = 0
    orig = L.sph_engine_substeps

    def slab_loop(Eref, half, full, nsub, stream):
        return L.sph_engine_substeps_slab(Eref, comm, ctypes.byref(P), half, full, nsub, stream)

    L.sph_engine_substeps = slab_loop
    try:
        sim = _sim(0.04)
        for _ in range(4):
            sim.advance()
    finally:
        L.sph_engine_substeps = orig
    for f in ("x", "v", "rho", "p", "drho", "dvdt", "nnb"):
        assert sim.registry.view(f).tobytes() == ref.registry.view(f).tobytes(), f
    assert sim.interaction_count == ref.interaction_count
    _native.check(L.sph_comm_destroy(comm), "destroy")

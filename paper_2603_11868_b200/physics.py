"""Weakly-compressible SPH on B200: kernel objects, bindings and the
device-resident step driver.

Mirror of ``minisph/physics.py``.  Host-side formulas (Wendland alpha, EOS,
``force_args`` scalars, time-step arithmetic) are the reference's own,
evaluated with the same NumPy-2 scalar rules so the device receives the
reference's exact binary32 scalars.  Every per-particle body runs in CUDA:
``CONTINUITY`` ... ``COPY_SCALAR`` dispatch by identity to the C ABI
(include/sph_b200.h), and :class:`Simulation` keeps the whole state in HBM
and runs ``advance`` as the fused engine of csrc/engine.cu.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
import time

import numpy as np

from . import _native
from . import variables as var
from ._device import (C_void, Staging, device_of, is_tensor, ptr, stream_ptr,
                      torch_mod, workspace)
from .execution import (ExecutionPolicy, ParticleKernel, ReduceSpec,
                        particle_for, particle_reduce)
from .neighborhood import (NEIGHBOR_CAPACITY, NeighborOverflowError,
                           build_cell_linked_list)


class SimulationUnstableError(RuntimeError):
    """physics.py:36-37"""


# -- smoothing kernel and EOS (physics.py:42-73), host scalars ---------------

def wendland_alpha(h, d):
    if d == 2:
        return 7.0 / (4.0 * math.pi * h * h)
    return 21.0 / (16.0 * math.pi * h ** 3)


def kernel_W(r, h, d):
    q = r / h
    if q >= 2.0:
        return 0.0
    t = 1.0 - 0.5 * q
    return wendland_alpha(h, d) * t ** 4 * (2.0 * q + 1.0)


def kernel_gradW(r, h, d):
    q = r / h
    if q >= 2.0:
        return 0.0
    t = 1.0 - 0.5 * q
    return -5.0 * wendland_alpha(h, d) * q * t ** 3 / h


def eos_pressure(rho, rho0, c0):
    return c0 * c0 * (rho - rho0)


def eos_density(p, rho0, c0):
    return rho0 + p / (c0 * c0)


# -- native kernel implementations (the particle_for boundary) ---------------

def _dtype_of(a):
    if is_tensor(a):
        return np.dtype(str(a.dtype).replace("torch.", ""))
    return np.asarray(a).dtype


def _fill_common(a, dtype, n, dim, origin, shape, cell_size, cutoff, h, alpha_d):
    dt = np.dtype(dtype).type
    for k in range(3):
        a.origin[k] = float(origin[k]) if k < dim else 0.0
        a.shape[k] = int(shape[k]) if k < dim else 1
    a.cell_size = dt(cell_size)
    a.cutoff = dt(cutoff)
    a.h = dt(h)
    a.alpha_d = dt(alpha_d)
    a.n = n
    a.dim = dim


def _run_sweep(entry, policy, n, fill):
    """Stage arrays, fill the SphSweepArgs struct, call, write back."""
    lib = _native.lib()
    dev = device_of(policy)
    with Staging(dev) as st:
        a, dtype = fill(st)
        ws_bytes = lib.sph_sweep_workspace_bytes(n)
        ws = workspace(dev, ws_bytes)
        fn = getattr(lib, f"sph_{entry}_{_native.sfx(dtype)}")
        rc = fn(ctypes.byref(a), ptr(ws), ws_bytes, stream_ptr(dev))
        _native.check(rc, entry)


def _force_sweep(entry, writes):
    """particle_for body for the force_args-bound sweeps (physics.py:94-194)."""

    def native(policy, n, args):
        (x, v, rho, p, m, wall, ids, g, offsets, pids, origin, shape,
         drho, dvdt, nnb, oflow, cell_size, cutoff, h, alpha_d, c0, rho0,
         avisc, eps_h2) = args
        dtype = _dtype_of(x)
        dim = int(np.asarray(shape).shape[0])

        def fill(st):
            a = _native.sweep_struct(dtype)()
            dev_arrays = {}
            for name, arr in (("x", x), ("v", v), ("rho", rho), ("p", p),
                              ("m", m), ("wall", wall), ("ids", ids),
                              ("offsets", offsets), ("pids", pids),
                              ("drho", drho), ("dvdt", dvdt), ("nnb", nnb),
                              ("oflow", oflow)):
                dev_arrays[name] = st.to_dev(arr, writeback=name in writes)
                setattr(a, name, ptr(dev_arrays[name]).value)
            _fill_common(a, dtype, n, dim, np.asarray(origin), np.asarray(shape),
                         cell_size, cutoff, h, alpha_d)
            gg = np.asarray(g)
            for k in range(3):
                a.g[k] = float(gg[k]) if k < dim else 0.0
            dt = np.dtype(dtype).type
            a.c0, a.rho0 = dt(c0), dt(rho0)
            a.alpha_visc, a.eps_h2 = dt(avisc), dt(eps_h2)
            return a, dtype

        _run_sweep(entry, policy, n, fill)

    return native


def _density_summation_native(policy, n, args):
    """physics.py:197-217 via its kernel-shell argument tuple (:376-380)."""
    (x, rho, m, ids, offsets, pids, origin, shape, cell_size, cutoff, h,
     alpha_d) = args
    dtype = _dtype_of(x)
    dim = int(np.asarray(shape).shape[0])

    def fill(st):
        a = _native.sweep_struct(dtype)()
        for name, arr, wb in (("x", x, False), ("rho", rho, True), ("m", m, False),
                              ("ids", ids, False), ("offsets", offsets, False),
                              ("pids", pids, False)):
            setattr(a, name, ptr(st.to_dev(arr, writeback=wb)).value)
        _fill_common(a, dtype, n, dim, np.asarray(origin), np.asarray(shape),
                     cell_size, cutoff, h, alpha_d)
        return a, dtype

    _run_sweep("density_summation", policy, n, fill)


def _shepard_native(policy, n, args):
    """physics.py:220-247 via the _shepard_filter tuple (:473-478)."""
    (x, rho, m, wall, ids, offsets, pids, origin, shape, rho_new, cell_size,
     cutoff, h, alpha_d) = args
    dtype = _dtype_of(x)
    dim = int(np.asarray(shape).shape[0])

    def fill(st):
        a = _native.sweep_struct(dtype)()
        for name, arr, wb in (("x", x, False), ("rho", rho, False), ("m", m, False),
                              ("wall", wall, False), ("ids", ids, False),
                              ("offsets", offsets, False), ("pids", pids, False),
                              ("rho_new", rho_new, True)):
            setattr(a, name, ptr(st.to_dev(arr, writeback=wb)).value)
        _fill_common(a, dtype, n, dim, np.asarray(origin), np.asarray(shape),
                     cell_size, cutoff, h, alpha_d)
        return a, dtype

    _run_sweep("shepard", policy, n, fill)


def _dim_of(vec):
    return int(vec.shape[1]) if len(vec.shape) == 2 else 1


def _integ_native(entry):
    def native(policy, n, args):
        lib = _native.lib()
        dev = device_of(policy)
        if entry in ("kick", "drift"):
            target, src, wall, scal = args
            dtype = _dtype_of(target)
            with Staging(dev) as st:
                t = st.to_dev(target, writeback=True)
                s_ = st.to_dev(src)
                w = st.to_dev(wall)
                fn = getattr(lib, f"sph_{entry}_{_native.sfx(dtype)}")
                rc = fn(ptr(t), ptr(s_), ptr(w), n, _dim_of(target),
                        np.dtype(dtype).type(scal), stream_ptr(dev))
                _native.check(rc, entry)
        elif entry == "density_update":
            rho, p, drho, wall, dt_, c0, rho0 = args
            dtype = _dtype_of(rho)
            T = np.dtype(dtype).type
            with Staging(dev) as st:
                r = st.to_dev(rho, writeback=True)
                pp = st.to_dev(p, writeback=True)
                d = st.to_dev(drho)
                w = st.to_dev(wall)
                fn = getattr(lib, f"sph_density_update_{_native.sfx(dtype)}")
                rc = fn(ptr(r), ptr(pp), ptr(d), ptr(w), n, T(dt_), T(c0), T(rho0),
                        stream_ptr(dev))
                _native.check(rc, entry)
        else:   # copy_scalar: dst[i] = src[i] for i < n
            dst, src = args
            with Staging(dev) as st:
                d = st.to_dev(dst, writeback=True)
                s_ = st.to_dev(src)
                nbytes = n * d.element_size() * (d[0].numel() if d.dim() > 1 else 1)
                rc = lib.sph_copy(ptr(d), ptr(s_), nbytes, stream_ptr(dev))
                _native.check(rc, entry)

    return native


def _vmax_native(policy, n, args):
    """VMAX_SPEC (physics.py:296-310): exact max of |row|, a float64."""
    (v,) = args
    lib = _native.lib()
    dev = device_of(policy)
    torch = torch_mod()
    dtype = _dtype_of(v)
    with Staging(dev) as st:
        vv = st.to_dev(v)
        out = st.empty((1,), torch.float64)
        fn = getattr(lib, f"sph_vmax_{_native.sfx(dtype)}")
        rc = fn(ptr(vv), n, _dim_of(v), ptr(out), stream_ptr(dev))
        _native.check(rc, "vmax")
        return np.float64(out.cpu().item())


def _body_doc(name):
    def body(i, args):   # pragma: no cover - documentation stub
        raise NotImplementedError(f"{name} runs on the GPU")
    body.__name__ = name
    return body


CONTINUITY = ParticleKernel(_body_doc("_continuity_body"), "continuity",
                            _force_sweep("continuity", {"drho", "oflow"}))
MOMENTUM = ParticleKernel(_body_doc("_momentum_body"), "momentum",
                          _force_sweep("momentum", {"dvdt", "nnb", "oflow"}))
WALL_PRESSURE = ParticleKernel(_body_doc("_wall_pressure_body"), "wall_pressure",
                               _force_sweep("wall_pressure",
                                            {"p", "rho", "nnb", "oflow"}))
DENSITY_SUMMATION = ParticleKernel(_body_doc("_density_summation_body"),
                                   "density_summation", _density_summation_native)
SHEPARD = ParticleKernel(_body_doc("_shepard_body"), "shepard", _shepard_native)
KICK = ParticleKernel(_body_doc("_kick_body"), "kick", _integ_native("kick"))
DRIFT = ParticleKernel(_body_doc("_drift_body"), "drift", _integ_native("drift"))
DENSITY_UPDATE = ParticleKernel(_body_doc("_density_update_body"), "density_update",
                                _integ_native("density_update"))
COPY_SCALAR = ParticleKernel(_body_doc("_copy_scalar_body"), "copy_scalar",
                             _integ_native("copy"))


def _vnorm_transform(i, args):   # pragma: no cover - documentation stub
    raise NotImplementedError("VMAX_SPEC runs on the GPU")


def _fmax(a, b):
    return max(a, b)


VMAX_SPEC = ReduceSpec(0.0, _vnorm_transform, _fmax, native=_vmax_native)


# -- kernel-shell layer (physics.py:315-381) ----------------------------------

def force_scalars(registry, grid):
    """The scalar tail of force_args with NumPy-2 scalar semantics
    (physics.py:327-330)."""
    dt = registry.dtype.type
    h = registry.singular("h")
    return (dt(grid.cell_size), dt(2.0 * h), dt(h),
            dt(wendland_alpha(h, registry.dim)),
            dt(registry.singular("c0")), dt(registry.singular("rho0")),
            dt(registry.singular("alpha_visc")), dt(0.01 * h * h))


def force_args(registry, cll):
    """The shared neighbour-sweep argument tuple (physics.py:315-330)."""
    return ((registry.view("x"), registry.view("v"), registry.view("rho"),
             registry.view("p"), registry.view("m"), registry.view("wall"),
             registry.view("id"), registry.singular("g"),
             cll.offsets, cll.particle_ids,
             cll.grid.origin.astype(registry.dtype),
             cll.grid.shape_array(),
             registry.view("drho"), registry.view("dvdt"),
             registry.view("nnb"), registry.view("oflow"))
            + force_scalars(registry, cll.grid))


def evaluate_forces(policy, registry, cll):
    evaluate_continuity(policy, registry, cll)
    evaluate_momentum(policy, registry, cll)


def evaluate_continuity(policy, registry, cll):
    particle_for(policy, registry.particle_count, CONTINUITY,
                 force_args(registry, cll))
    _check_overflow(registry)


def evaluate_momentum(policy, registry, cll):
    particle_for(policy, registry.particle_count, MOMENTUM,
                 force_args(registry, cll))
    _check_overflow(registry)


def extrapolate_wall_pressure(policy, registry, cll):
    particle_for(policy, registry.particle_count, WALL_PRESSURE,
                 force_args(registry, cll))
    _check_overflow(registry)


def _check_overflow(registry):
    if registry.view("oflow").any():
        raise NeighborOverflowError(
            f"neighbor buffer capacity {NEIGHBOR_CAPACITY} exceeded")


class DensitySummationDynamics:
    """rho_i = sum_j m_j W_ij including self (physics.py:363-381)."""

    kernel = DENSITY_SUMMATION

    def __init__(self, registry, cll):
        self.registry = registry
        self.cll = cll

    def setup(self):
        reg, cll = self.registry, self.cll
        dt = reg.dtype.type
        h = reg.singular("h")
        args = (reg.view("x"), reg.view("rho"), reg.view("m"), reg.view("id"),
                cll.offsets, cll.particle_ids,
                cll.grid.origin.astype(reg.dtype), cll.grid.shape_array(),
                dt(cll.grid.cell_size), dt(2.0 * h), dt(h),
                dt(wendland_alpha(h, reg.dim)))
        return reg.particle_count, args


# -- time stepping (physics.py:386-413) --------------------------------------

def timestep_formula(vmax, amax, h, c0, dt_max, cfl_acoustic=0.6,
                     cfl_advective=0.25):
    """The host arithmetic of compute_timestep (physics.py:392-400)."""
    dt_acoustic = cfl_acoustic * h / (c0 + vmax)
    dt_advective = dt_max
    if vmax > 0.0:
        dt_advective = min(dt_advective, cfl_advective * h / vmax)
    if amax > 0.0:
        dt_advective = min(dt_advective, cfl_advective * math.sqrt(h / amax))
    return dt_acoustic, dt_advective


def compute_timestep(policy, registry, dt_max, cfl_acoustic=0.6,
                     cfl_advective=0.25):
    """Dual criteria from exact device max-reductions (physics.py:386-400)."""
    n = registry.particle_count
    vmax = float(particle_reduce(policy, n, VMAX_SPEC, (registry.view("v"),)))
    amax = float(particle_reduce(policy, n, VMAX_SPEC, (registry.view("dvdt"),)))
    return timestep_formula(vmax, amax, float(registry.singular("h")),
                            float(registry.singular("c0")), dt_max,
                            cfl_acoustic, cfl_advective)


def setup_state_variables(registry):
    """physics.py:403-413"""
    for name, kind in (("x", var.VECTOR), ("v", var.VECTOR),
                       ("rho", var.SCALAR), ("p", var.SCALAR),
                       ("m", var.SCALAR), ("Vol", var.SCALAR),
                       ("drho", var.SCALAR), ("dvdt", var.VECTOR),
                       ("rho_scratch", var.SCALAR)):
        registry.register_discrete(name, kind)
    registry.register_discrete("wall", var.INDEX)
    registry.register_discrete("nnb", var.INDEX)
    registry.register_discrete("oflow", var.INDEX)


# -- device-resident driver ----------------------------------------------------

SUBSTEP_KERNELS = ("kick_drift", "list_filter", "continuity_du", "wall_pressure",
                   "momentum_kick")

_ENGINE_FIELDS = ("x", "v", "rho", "p", "m", "Vol", "drho", "dvdt",
                  "rho_scratch", "id", "wall", "nnb", "oflow")
# fields the engine never writes (oflow: only on overflow, which is tracked)
_HOST_SAME_FIELDS = ("m", "Vol", "id", "wall", "oflow", "rho_scratch")
# the two halves of an overlapped push (sph_engine_push_begin / _end): the
# fields that place the particles, then the rest
_PUSH_FIRST = ("x", "id", "wall")
_PUSH_REST = ("v", "rho", "p", "m", "Vol", "drho", "dvdt", "rho_scratch", "nnb", "oflow")
# by-id fields the step itself never reads (rho_scratch: except on a Shepard
# step): uploaded last and delivered after the sub-steps (sph_engine_push_tail)
_PUSH_TAIL = ("Vol", "rho_scratch", "oflow")
# a step that starts from a host push uploads the second half behind its own
# skin-list build (SPH_PUSH_OVERLAP=0: the plain push)
PUSH_OVERLAP = os.environ.get("SPH_PUSH_OVERLAP", "1") != "0"
# ... and a step whose result was viewed after each of the last two steps
# pulls it within the step, overlapping the D2H copies with the last
# sub-step's sweeps (SPH_EAGER_PULL=0: pulls on view only)
EAGER_PULL = os.environ.get("SPH_EAGER_PULL", "1") != "0"
# registry fields by the engine event after which the step's values are final
_PULL_AT_X = ("x",)
_PULL_AT_RP = ("rho", "p", "drho")


def _key_to_double(k):
    """Inverse of the kernels' order-preserving double -> u64 key."""
    if k & (1 << 63):
        u = k & ~(1 << 63)
    else:
        u = ~k & 0xFFFFFFFFFFFFFFFF
    return struct.unpack("<d", struct.pack("<Q", u))[0]


def _bits_to_double(b):
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def engine_alloc(dev, n_cap, nf_cap, nw_cap, d, f64, grid, scalars, g, id_range=0,
                 persist=True):
    """Device storage of one engine (include/sph_b200.h SphEngine) for up to
    n_cap particles of which at most nf_cap fluid and nw_cap wall (the list
    tiles of the two segments are sized separately).  Returns the struct and
    the torch tensors backing it; engine_set_counts sets the live sizes."""
    torch = torch_mod()
    tdt = torch.float64 if f64 else torch.float32
    i32 = torch.int32
    ncells = grid.cell_count
    lib = _native.lib()
    n = max(int(n_cap), 1)
    nid = max(n, int(id_range))     # by-id arrays (global ids on slab ranks)
    tiles = max((nf_cap + 31) // 32 + (nw_cap + 31) // 32, 1)
    T = {}
    for k in ("pos0", "pos1", "vel0", "vel1", "dvdt"):
        T[k] = torch.empty((n, 4), dtype=tdt, device=dev)
    for k in ("rp0", "rp1", "rq"):
        T[k] = torch.empty((n, 2), dtype=tdt, device=dev)
    for k in ("drho", "disp", "disp0"):
        T[k] = torch.empty((n,), dtype=tdt, device=dev)
    for k in ("rho_scratch_id", "vol_id"):
        T[k] = torch.empty((nid,), dtype=tdt, device=dev)
    for k in ("id", "nnb", "refpos", "cell0", "queue"):
        T[k] = torch.empty((n,), dtype=i32, device=dev)
    for k in ("oflow_id", "wall_id"):
        T[k] = torch.empty((nid,), dtype=i32, device=dev)
    T["owned_id"] = torch.ones((nid,), dtype=torch.uint8, device=dev)
    T["offs_f"] = torch.empty((ncells + 1,), dtype=i32, device=dev)
    T["offs_w"] = torch.empty((ncells + 1,), dtype=i32, device=dev)
    T["lists"] = torch.empty((tiles, NEIGHBOR_CAPACITY, 32), dtype=i32, device=dev)
    if persist:   # skin lists carried across steps (sph_engine_maintain_lists)
        T["lists_alt"] = torch.empty((tiles, NEIGHBOR_CAPACITY, 32), dtype=i32, device=dev)
        T["lcount_alt"] = torch.empty((tiles * 32,), dtype=i32, device=dev)
        for k in ("key_sorted", "key_prev", "perm", "inv"):
            T[k] = torch.empty((n,), dtype=i32, device=dev)
        if not f64:   # local displacement bounds (csrc engine.cu k_blockmax)
            for k in ("cellmax", "blockmax"):
                T[k] = torch.zeros((max(ncells, 1),), dtype=i32, device=dev)
    T["elist"] = torch.empty((tiles, NEIGHBOR_CAPACITY, 32), dtype=i32, device=dev)
    for k in ("lcount", "acount", "nww"):
        T[k] = torch.empty((tiles * 32,), dtype=i32, device=dev)
    T["qcount"] = torch.zeros((4,), dtype=i32, device=dev)
    ws_bytes = lib.sph_engine_workspace_bytes_ids(n, ncells, int(f64), int(id_range))
    T["ws"] = torch.empty((ws_bytes,), dtype=torch.uint8, device=dev)
    T["stats"] = torch.zeros((ctypes.sizeof(_native.SphStepStats),), dtype=torch.uint8,
                             device=dev)
    E = _native.SphEngine()
    E.ncells, E.dim = ncells, d
    E.key_bits = max(1, int(ncells - 1).bit_length())
    E.pos[0], E.pos[1] = T["pos0"].data_ptr(), T["pos1"].data_ptr()
    E.vel[0], E.vel[1] = T["vel0"].data_ptr(), T["vel1"].data_ptr()
    E.rp[0], E.rp[1] = T["rp0"].data_ptr(), T["rp1"].data_ptr()
    E.rq = T["rq"].data_ptr()
    for k in ("dvdt", "drho", "id", "nnb", "refpos", "rho_scratch_id",
              "oflow_id", "wall_id", "vol_id", "offs_f", "offs_w", "lists",
              "lcount", "acount", "nww", "elist", "cell0", "disp", "disp0", "queue",
              "qcount", "ws", "stats"):
        setattr(E, k, T[k].data_ptr())
    E.owned_id = None      # every particle owned (multi-rank runs set it)
    E.id_range = int(id_range)
    for k in ("lists_alt", "lcount_alt", "key_sorted", "key_prev", "perm", "inv", "cellmax",
              "blockmax"):
        setattr(E, k, T[k].data_ptr() if k in T else None)
    E.ws_bytes = ws_bytes
    (cs, cutoff, h, alpha_d, c0, rho0, avisc, eps_h2) = scalars
    g = np.asarray(g)
    origin = grid.origin.astype(np.float64 if f64 else np.float32)
    for k in range(3):
        E.g[k] = float(g[k]) if k < d else 0.0
        E.origin[k] = float(origin[k]) if k < d else 0.0
        E.shape[k] = int(grid.shape[k]) if k < d else 1
    E.cell_size, E.cutoff, E.h, E.alpha_d = float(cs), float(cutoff), float(h), float(alpha_d)
    E.c0, E.rho0, E.alpha_visc, E.eps_h2 = float(c0), float(rho0), float(avisc), float(eps_h2)
    E.f64 = int(f64)
    per = getattr(grid, "period", None)
    for k in range(3):   # periodic box (run-precision periods; 0 = bounded)
        E.period[k] = float((np.float64 if f64 else np.float32)(per[k])) \
            if per is not None and k < d else 0.0
    return E, T


# Verlet skin = factor x (vmax dt + amax dt^2) + 0.02 cutoff, the factor
# adapted per step from the displacement-triggered refreshes (experiment
# overrides through the environment)
SKIN_FACTOR_START = float(os.environ.get("SPH_SKIN_START", "2.0"))
SKIN_FACTOR_FLOOR = float(os.environ.get("SPH_SKIN_FLOOR", "0.5"))
SKIN_MARGIN = float(os.environ.get("SPH_SKIN_MARGIN", "0.02"))


# Skin lists kept across advective steps (epochs): the skin is sized for
# LIST_EPOCH_STEPS steps of displacement; an epoch ends (full rebuild) when
# the largest displacement since its build passes LIST_EPOCH_LIMIT x skin.
LIST_EPOCH_STEPS = int(os.environ.get("SPH_LIST_EPOCH_STEPS", "3"))
LIST_EPOCH_LIMIT = float(os.environ.get("SPH_LIST_EPOCH_LIMIT", "0.8"))
# an epoch that carried no step backs off for this many steps (its wider
# skin only cost sweep work)
LIST_EPOCH_BACKOFF = int(os.environ.get("SPH_LIST_EPOCH_BACKOFF", "8"))
# with local displacement bounds: carry while the last step refreshed at most
# this fraction of the lists per sub-step, for at most LIST_EPOCH_MAX steps
LIST_EPOCH_REFRESH = float(os.environ.get("SPH_LIST_EPOCH_REFRESH", "0.002"))
LIST_EPOCH_MAX = int(os.environ.get("SPH_LIST_EPOCH_MAX", "6"))


def grid_is_periodic(grid):
    per = getattr(grid, "period", None)
    return per is not None and any(float(p) > 0.0 for p in per)


def engine_set_counts(E, n, nf):
    E.n, E.nf = int(n), int(nf)


def _upload_async(arr, device):
    """Host registry field -> device tensor, queued on the current stream
    (asynchronous from pinned memory; a pageable source is staged by the
    driver before the call returns)."""
    torch = torch_mod()
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device, non_blocking=True)


class Simulation:
    """Advective-step driver (physics.py:416-564) with the state in HBM.

    Constructor, attributes and methods follow the reference.  The registry
    stays the user-facing owner: the first ``initialize``/``advance`` pushes
    it to the device; ``registry.view(...)`` pulls the device state back into
    the registry's arrays in the reference's physical order (the engine tracks
    the reference's sort_every permutation), after which the host copy is
    authoritative again for the next step.
    """

    def __init__(self, registry, grid, policy, dt_max=1e-3, sort_every=100,
                 shepard_every=200, fixed_dt=None, cfl_acoustic=0.6,
                 cfl_advective=0.25):
        self.registry = registry
        self.grid = grid
        self.policy = policy
        self.dt_max = dt_max
        self.sort_every = sort_every
        self.shepard_every = shepard_every
        self.fixed_dt = fixed_dt
        self.cfl_acoustic = cfl_acoustic
        self.cfl_advective = cfl_advective
        self.step_count = 0
        self.time = 0.0
        self.interaction_count = 0
        self.phase_seconds = {"cll": 0.0, "interactions": 0.0,
                              "integration": 0.0, "sorting": 0.0}
        self.out_of_bounds = 0
        self.last_nsub = 0
        self._dev = None
        self._host_dirty = True     # host registry is authoritative
        self._host_stale = False    # device is ahead of the host registry
        # fields whose host copy still equals the device's (the engine never
        # writes them and the registry order has not changed since the push):
        # a pull skips their device -> host copies
        self._host_same = set()
        self._norms = None          # (vmax, amax) valid for the device state
        self.last_push_bytes = 0
        self.last_pull_bytes = 0
        self._oob_walls = 0
        self.kernel_times = None    # dict name -> [ms per launch] when profiling
        self._pending_events = []
        self._skin_factor = SKIN_FACTOR_START
        self.last_nfix = 0
        self.list_refresh = "auto"  # sub-step list upkeep: auto | pass | queue
        # skin lists carried across steps: "auto" (3D, when the skin allows
        # it), "always" (any dimension; tests) or "off" (rebuilt every step: the default -- measured on the
        # dam break, the carried steps save list builds but the displacement
        # test against the GLOBAL largest displacement then refreshes many
        # lists per sub-step, profiles/r02/ab)
        self.list_epochs = os.environ.get("SPH_LIST_EPOCHS", "off")
        self._epoch = None          # (skin, steps) of the lists' epoch
        self._epoch_backoff = 0     # steps left without epochs after a futile one
        self.last_list_mode = None  # "build" | "maintain" (diagnostic)
        self._last_step = None      # (vmax, amax, dt) of the last step: skin forecast
        self.push_overlap = PUSH_OVERLAP
        self.last_push_overlapped = False
        self._pending_tail = None   # (event, {field: landing tensor}) of a split push
        self.eager_pull = EAGER_PULL
        self.last_pull_overlapped = False
        self._viewed = False        # a registry view since the last step
        self._view_streak = 0       # consecutive steps followed by a view
        registry.attach_engine(self)

    def _lib(self):
        """libsphb200.so, or its periodic-box build for a periodic grid."""
        return _native.lib(periodic=grid_is_periodic(self.grid))

    # -- registry coupling ----------------------------------------------------

    def host_modified(self):
        self._host_dirty = True
        self._norms = None

    def pull_to_host(self):
        """Write the device state into the registry (reference order)."""
        self._viewed = True
        if self._dev is None:
            return
        if not self._host_stale:
            if not self._host_dirty:
                # the step already pulled its result (_pull_overlapped): the
                # host copy is current, and from now on the caller may edit it
                self._host_dirty = True
                self._host_same = set()
                self._norms = None
            return
        self._host_stale = False
        d = self._dev
        torch = torch_mod()
        reg = self.registry
        outs = {}
        with torch.cuda.stream(d["tstream"]):
            for f in _ENGINE_FIELDS:
                host = reg.raw_view(f)
                tdt = torch.int32 if host.dtype == np.uint32 else d["tdtype"]
                outs[f] = torch.empty(host.shape, dtype=tdt, device=d["device"])
            rc = self._lib().sph_engine_pull(
                ctypes.byref(d["E"]), *[ptr(outs[f]) for f in _ENGINE_FIELDS],
                d["stream"])
            _native.check(rc, "engine_pull")
            self.last_pull_bytes = 0
            for f in _ENGINE_FIELDS:   # queued back to back, one synchronise
                if f in self._host_same:
                    continue
                host = reg.raw_view(f)
                self.last_pull_bytes += host.nbytes
                hv = host.view(np.int32) if host.dtype == np.uint32 else host
                torch.from_numpy(hv).copy_(outs[f], non_blocking=True)
        d["tstream"].synchronize()
        # the caller may now modify the host arrays in place
        self._host_dirty = True
        self._host_same = set()
        self._norms = None

    @property
    def cll(self):
        """A reference CellLinkedList of the current positions (diagnostic)."""
        return build_cell_linked_list(self.policy, self.registry.view("x"),
                                      self.grid)

    # -- device state ---------------------------------------------------------

    def _alloc(self, nf=None):
        reg = self.registry
        if self.grid.dim != reg.dim:
            raise ValueError("grid and registry dimensions differ")
        if nf is None:
            nf = int((reg.raw_view("wall") == 0).sum())
        n = reg.particle_count
        E, T = engine_alloc(device_of(self.policy), n, nf, n - nf, reg.dim,
                            reg.dtype == np.float64, self.grid,
                            force_scalars(reg, self.grid), reg.singular("g"),
                            persist=self.list_epochs != "off")
        engine_set_counts(E, n, nf)
        torch = torch_mod()
        # the engine's stream: every engine call and every copy to or from
        # its buffers is queued on it, whatever stream is current later
        tstream = torch.cuda.current_stream(T["pos0"].device)
        self._dev = {"device": T["pos0"].device, "E": E, "T": T, "tdtype": T["pos0"].dtype,
                     "tstream": tstream, "stream": C_void(tstream.cuda_stream),
                     "stats_host": torch.empty(T["stats"].shape, dtype=torch.uint8,
                                               pin_memory=True),
                     "cstream": None}   # upload stream of overlapped pushes (lazy)

    def _push(self, devs=None, nf=None):
        """Registry -> device SoA (physics layout, cell order)."""
        reg = self.registry
        if self._dev is None:
            self._alloc(nf)
        d = self._dev
        st = Staging(d["device"])
        host_push = devs is None
        if devs is None:
            # every field's upload is queued on the engine's stream before the
            # push kernels (pinned registries copy asynchronously; the
            # stats read below synchronises before the host may touch them)
            with torch_mod().cuda.stream(d["tstream"]):
                devs = [_upload_async(reg.raw_view(f), d["device"]) for f in _ENGINE_FIELDS]
            self.last_push_bytes = sum(reg.raw_view(f).nbytes for f in _ENGINE_FIELDS)
        else:   # caller-provided device tensors: ordered before the push
            d["tstream"].wait_stream(torch_mod().cuda.current_stream(d["device"]))
        # the id-permutation check and the fluid count run on the device
        for attempt in range(2):
            rc = self._lib().sph_engine_push(ctypes.byref(d["E"]),
                                               *[ptr(t) for t in devs], d["stream"])
            _native.check(rc, "engine_push")
            stats = self._read_stats()
            if stats.push_error:
                raise ValueError("registry ids must be a permutation of 0..N-1")
            if stats.fluid_seen == d["E"].nf or attempt:
                break
            self._alloc(int(stats.fluid_seen))   # the wall flags changed: resize
            d = self._dev
        self._oob_walls = stats.oob_walls
        # the host arrays now hold what the device holds; the engine never
        # writes m, Vol, id, wall (nor oflow / rho_scratch outside overflow /
        # Shepard), so those stay equal until the registry order changes
        self._host_same = set(_HOST_SAME_FIELDS) if host_push else set()
        del devs, st
        self._host_dirty = False
        self._host_stale = False
        self._norms = None

    def _overlap_ready(self):
        """A host push can be split around the step's list build: the
        device is allocated for this registry, the previous step's norms and
        dt forecast the skin (the skin affects speed only: csrc/engine.cu
        rebuilds any list a particle outruns), and lists are rebuilt every
        step (no epochs)."""
        d = self._dev
        if not (self.push_overlap and self._host_dirty and d is not None and self._last_step
                and self.list_epochs == "off"):
            return False
        reg = self.registry
        return d["E"].n == reg.particle_count and d["E"].nf > 0

    def _push_overlapped(self):
        """Host push in two halves around this step's list build: x, id and
        wall are uploaded and placed (sph_engine_push_begin: cell order, the
        CLL of this step) while the other ten fields are still in
        flight on a copy stream; the skin lists are built from the placed
        positions with the forecast skin; sph_engine_push_end gathers the
        rest once it has landed.  Nothing synchronises here: the step's
        first stats read checks the push (push_error / fluid_seen)."""
        torch = torch_mod()
        d = self._dev
        reg = self.registry
        ts = d["tstream"]
        cs = self._copy_stream()
        ev_first, ev_rest, ev_tail = d["push_events"]
        shepard = self.shepard_every and self.step_count > 0 \
            and self.step_count % self.shepard_every == 0
        tail = tuple(f for f in _PUSH_TAIL if not (shepard and f == "rho_scratch"))

        def upload(f):
            src = self._host_tensor(f)
            dst = self._landing(f, src)
            dst.copy_(src, non_blocking=True)
            return dst

        cs.wait_stream(ts)   # the last push's landing buffers are consumed
        with torch.cuda.stream(cs):
            first = [upload(f) for f in _PUSH_FIRST]
            ev_first.record(cs)
            rest = {f: upload(f) for f in _PUSH_REST if f not in tail}
            ev_rest.record(cs)
            late = {f: upload(f) for f in tail}
            ev_tail.record(cs)
        self.last_push_bytes = sum(reg.raw_view(f).nbytes for f in _ENGINE_FIELDS)
        ts.wait_event(ev_first)
        rc = self._lib().sph_engine_push_begin(ctypes.byref(d["E"]),
                                               *[ptr(t) for t in first], d["stream"])
        _native.check(rc, "engine_push_begin")
        vmax, amax, dt = self._last_step
        t0 = time.perf_counter()
        with self._kernel_event("skin_build"):
            self._build_lists(self._choose_skin(vmax, amax, dt))
        self.last_list_mode = "build"
        self.phase_seconds["cll"] += time.perf_counter() - t0
        ts.wait_event(ev_rest)
        rc = self._lib().sph_engine_push_end(
            ctypes.byref(d["E"]), *[ptr(rest[f]) if f in rest else None for f in _PUSH_REST],
            d["stream"])
        _native.check(rc, "engine_push_end")
        late["id"] = first[_PUSH_FIRST.index("id")]
        self._pending_tail = (ev_tail, late)
        self._host_same = set(_HOST_SAME_FIELDS)
        self._host_dirty = False
        self._host_stale = False
        self._norms = None

    def _deliver_tail(self):
        """Queue the deferred by-id fields of the last split push (after the
        step's sub-steps: nothing before reads them)."""
        if self._pending_tail is None:
            return
        ev, late = self._pending_tail
        self._pending_tail = None
        d = self._dev
        d["tstream"].wait_event(ev)
        rc = self._lib().sph_engine_push_tail(
            ctypes.byref(d["E"]), ptr(late["id"]),
            *[ptr(late[f]) if f in late else None for f in _PUSH_TAIL], d["stream"])
        _native.check(rc, "engine_push_tail")

    def _copy_stream(self):
        """The engine's host-transfer stream, its events and its device
        landing buffers (registry layout, reused by every overlapped push
        and pull; created on first use)."""
        torch = torch_mod()
        d = self._dev
        if d["cstream"] is None:
            d["cstream"] = torch.cuda.Stream(device=d["device"])
            d["landing"] = {}
            d["push_events"] = (torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event())
            ev = [torch.cuda.Event() for _ in range(3)]
            for e in ev:   # materialise the events: their handles go to the library
                e.record(d["tstream"])
            d["pull_events"] = ev
        return d["cstream"]

    def _host_tensor(self, f):
        a = np.ascontiguousarray(self.registry.raw_view(f))
        if a.dtype == np.uint32:
            a = a.view(np.int32)
        return torch_mod().from_numpy(a)

    def _landing(self, f, like):
        d = self._dev
        dst = d["landing"].get(f)
        if dst is None or dst.shape != like.shape or dst.dtype != like.dtype:
            dst = d["landing"][f] = torch_mod().empty(like.shape, dtype=like.dtype,
                                                      device=d["device"])
        return dst

    def _eager_pull_ready(self):
        """Pull this step's result within the step: the result of each of
        the last two steps was viewed, and the registry is in contiguous
        pinned host memory (a pageable copy would block the host mid-step)."""
        if not (self.eager_pull and self._viewed and self._view_streak >= 1
                and self.kernel_times is None and self.registry.particle_count):
            return False
        reg = self.registry
        return all(reg.raw_view(f).flags.c_contiguous and self._host_tensor(f).is_pinned()
                   for f in _ENGINE_FIELDS)

    def _pull_overlapped(self, marks, ev_end):
        """Queue the step's registry pull on the copy stream: x once the last
        sub-step's positions are final, rho / p / drho after its wall
        sweep (both during the momentum sweep), the rest after the step;
        fields the host provably still holds (_host_same) are skipped."""
        torch = torch_mod()
        d = self._dev
        cs = self._copy_stream()
        late = tuple(f for f in _ENGINE_FIELDS
                     if f not in _PULL_AT_X + _PULL_AT_RP and f not in self._host_same)
        lib = self._lib()
        nbytes = 0
        with torch.cuda.stream(cs):
            for ev, fields in ((marks[0], _PULL_AT_X), (marks[1], _PULL_AT_RP),
                               (ev_end, late)):
                cs.wait_event(ev)
                hosts = {f: self._host_tensor(f) for f in fields}
                lands = {f: self._landing(f, hosts[f]) for f in fields}
                mask = sum(1 << _ENGINE_FIELDS.index(f) for f in fields)
                args = [ptr(lands[f]) if f in lands else None for f in _ENGINE_FIELDS]
                rc = lib.sph_engine_pull_fields(ctypes.byref(d["E"]), mask, *args,
                                                C_void(cs.cuda_stream))
                _native.check(rc, "engine_pull_fields")
                for f in fields:
                    hosts[f].copy_(lands[f], non_blocking=True)
                    nbytes += hosts[f].numel() * hosts[f].element_size()
        self.last_pull_bytes = nbytes

    def load_device_state(self, state):
        """Start from registry-order device tensors (``cases.build_case_device``;
        the fields of the registry, uint32 ones as int32) instead of the host
        registry: the engine becomes authoritative and the host registry is
        filled only when a view is requested."""
        n = self.registry.particle_count
        devs = []
        for f in _ENGINE_FIELDS:
            t = state[f]
            shape = self.registry.raw_view(f).shape
            if tuple(t.shape) != tuple(shape) or not t.is_cuda or not t.is_contiguous():
                raise TypeError(f"device state field {f!r}: expected a contiguous "
                                f"CUDA tensor of shape {shape}")
            devs.append(t)
        nf = int((state["wall"] == 0).sum().item()) if n else 0
        if self._dev is not None and self._dev["device"] != devs[0].device:
            raise TypeError("device state lives on another device")
        self._push(devs, nf)
        self._host_stale = True     # the host registry has not seen this state

    def _ensure_device(self):
        if self._host_dirty:
            self._push()

    def _call(self, name, *args):
        d = self._dev
        rc = getattr(self._lib(), name)(ctypes.byref(d["E"]), *args, d["stream"])
        _native.check(rc, name)

    def _read_stats(self):
        d = self._dev
        with torch_mod().cuda.stream(d["tstream"]):
            d["stats_host"].copy_(d["T"]["stats"], non_blocking=True)
        d["tstream"].synchronize()
        return _native.SphStepStats.from_buffer_copy(d["stats_host"].numpy().tobytes())

    def _finish_counts(self, stats, check):
        if stats.overflow:   # the sweeps flagged oflow of some particles
            self._host_same.discard("oflow")
        if stats.overflow and check:
            raise NeighborOverflowError(
                f"neighbor buffer capacity {NEIGHBOR_CAPACITY} exceeded")
        self._norms = (_bits_to_double(stats.vmax_bits),
                       _bits_to_double(stats.amax_bits))

    # -- reference API ---------------------------------------------------------

    def _rebuild_cll(self):
        """physics.py:446-449 on the engine layout."""
        t0 = time.perf_counter()
        with self._kernel_event("cll_rebuild"):
            self._call("sph_engine_rebuild_cll")
        self.phase_seconds["cll"] += time.perf_counter() - t0

    def _kernel_event(self, name):
        """CUDA events on the engine stream around a per-step part when
        kernel_times is set (read, without an extra synchronisation, after
        the step's stats read)."""
        sim = self

        class _Ev:
            def __enter__(self_):
                if sim.kernel_times is None:
                    return self_
                torch = torch_mod()
                self_.e = (torch.cuda.Event(enable_timing=True),
                           torch.cuda.Event(enable_timing=True))
                self_.e[0].record(sim._dev["tstream"])
                return self_

            def __exit__(self_, *exc):
                if sim.kernel_times is not None and hasattr(self_, "e"):
                    self_.e[1].record(sim._dev["tstream"])
                    sim._pending_events.append((name, self_.e))
                return False
        return _Ev()

    def _collect_events(self):
        for name, (e0, e1) in self._pending_events:
            e1.synchronize()
            self.kernel_times.setdefault(name, []).append(e0.elapsed_time(e1))
        self._pending_events = []

    def initialize(self):
        """physics.py:460-467: CLL, wall pressure, momentum, counts."""
        self._ensure_device()
        self._call("sph_engine_stats", ctypes.c_int32(_native.STATS_RESET))
        self._rebuild_cll()
        t0 = time.perf_counter()
        self._build_lists(0.0)
        self._call("sph_engine_initialize")
        self._call("sph_engine_stats", ctypes.c_int32(_native.STATS_NORMS))
        stats = self._read_stats()
        self.phase_seconds["interactions"] += time.perf_counter() - t0
        self._host_stale = True
        self.out_of_bounds += stats.oob + self._oob_walls
        self._finish_counts(stats, check=True)
        self.interaction_count += int(stats.interactions)

    def _shepard_filter(self):
        """physics.py:469-487 (SHEPARD, COPY_SCALAR, DENSITY_UPDATE(0))."""
        self._ensure_device()
        self._build_lists(0.0)
        self._call("sph_engine_shepard")
        self._host_same.discard("rho_scratch")
        self._host_stale = True

    def _build_lists(self, skin):
        """Ascending-id Verlet lists within cutoff + skin (csrc/engine.cu)."""
        self._call("sph_engine_build_lists", ctypes.c_double(skin))
        self._epoch = None

    def _lists_for_step(self, vmax, amax, dt):
        """This step's skin lists: carried over from the previous step
        (sph_engine_maintain_lists) while the epoch's skin still covers the
        displacement, else built afresh.  An epoch's skin is sized for
        LIST_EPOCH_STEPS steps; where that would pass the skin cap (fast
        flows) every step rebuilds, as before."""
        E = self._dev["E"]
        cutoff = float(E.cutoff)
        est = vmax * dt + amax * dt * dt
        cap = (0.45 if self.registry.dim == 3 else 1.0) * cutoff
        per_step = self._skin_factor * est
        ep = self._epoch
        auto = (self.list_epochs == "auto" and self.registry.dim == 3) or \
            self.list_epochs == "always"
        if ep is not None and E.cellmax is not None:
            # local bounds: a list fails only where its own block moved; carry
            # while the last step refreshed few lists
            carry = (ep["refresh"] <= LIST_EPOCH_REFRESH and ep["steps"] < LIST_EPOCH_MAX)
        else:
            carry = ep is not None and ep["dmax"] + per_step <= LIST_EPOCH_LIMIT * ep["skin"]
        if ep is not None and E.lists_stale and auto and carry:
            self._call("sph_engine_maintain_lists")
            ep["steps"] += 1
            self.last_list_mode = "maintain"
            return
        if ep is not None and ep["steps"] == 1:   # the epoch carried nothing
            self._epoch_backoff = LIST_EPOCH_BACKOFF
        elif self._epoch_backoff > 0:
            self._epoch_backoff -= 1
        # 2D lists are cheap next to a 2D step's many sub-steps: no epochs
        k = LIST_EPOCH_STEPS if auto and self._epoch_backoff == 0 else 1
        skin = min(k * per_step + SKIN_MARGIN * cutoff, cap)
        if k > 1 and (skin >= cap or E.key_sorted is None):
            skin, k = self._choose_skin(vmax, amax, dt), 1
        self._build_lists(skin)
        self.last_list_mode = "build"
        if k > 1:
            self._epoch = {"skin": skin, "steps": 1, "dmax": 0.0, "refresh": 0.0}

    def _choose_skin(self, vmax, amax, dt):
        """Skin for this step's lists: a multiple of the displacement the
        step's own dt allows; any particle that outruns it is rebuilt exactly
        on the device, so the choice affects speed only."""
        cutoff = float(self._dev["E"].cutoff)
        est = vmax * dt + amax * dt * dt
        cap = (0.45 if self.registry.dim == 3 else 1.0) * cutoff
        return min(self._skin_factor * est + SKIN_MARGIN * cutoff, cap)

    def _adapt_skin(self, ndisp, nsub):
        """Grow the skin when displacement-triggered refreshes are frequent,
        shrink it towards the 2x-displacement floor otherwise (refreshes
        after a cell change do not depend on the skin)."""
        n = max(1, self.registry.particle_count)
        frac = ndisp / (n * max(1, nsub))
        if frac > 2e-3:
            self._skin_factor = min(self._skin_factor * 1.5, 16.0)
        elif frac < 5e-4:
            self._skin_factor = max(SKIN_FACTOR_FLOOR, self._skin_factor * 0.95)

    def advance(self, end_time=None):
        """One advective step (physics.py:489-552); returns the dt taken."""
        overlapped = self._overlap_ready()
        if overlapped:
            # the push's cell order is this step's CLL (the rebuild would
            # re-sort an already sorted layout: identity) and its clamp count
            self._push_overlapped()
        else:
            self._ensure_device()
        self.last_push_overlapped = overlapped
        d = self._dev
        L = self._lib()
        if self.sort_every and self.step_count > 0 \
                and self.step_count % self.sort_every == 0:
            t0 = time.perf_counter()
            self._call("sph_engine_ref_sort")
            self._host_same = set()      # the registry order changed
            self.phase_seconds["sorting"] += time.perf_counter() - t0
        if overlapped:   # counters were zeroed by the push
            self._call("sph_engine_stats", ctypes.c_int32(_native.STATS_NORMS))
        else:
            flags = _native.STATS_RESET | (0 if self._norms else _native.STATS_NORMS)
            self._call("sph_engine_stats", ctypes.c_int32(flags))
            self._rebuild_cll()
        # compute_timestep (physics.py:502-511) reads only v and dvdt, which the
        # Shepard filter does not touch, so the step's dt is known before the
        # lists are built and sizes their skin
        t0 = time.perf_counter()
        if self._norms is None:
            s = self._read_stats()
            if overlapped:
                if s.push_error:
                    self._host_dirty = True
                    self._pending_tail = None
                    raise ValueError("registry ids must be a permutation of 0..N-1")
                if s.fluid_seen != d["E"].nf:   # the wall flags changed: plain push
                    self._host_dirty = True
                    self._pending_tail = None
                    self._last_step = None
                    return self.advance(end_time)
                self._oob_walls = s.oob_walls
            self._norms = (_bits_to_double(s.vmax_bits), _bits_to_double(s.amax_bits))
        vmax, amax = self._norms
        if self.fixed_dt is not None:
            dt_ac = dt_adv = self.fixed_dt
        else:
            dt_ac, dt_adv = timestep_formula(
                vmax, amax, float(self.registry.singular("h")),
                float(self.registry.singular("c0")), self.dt_max,
                self.cfl_acoustic, self.cfl_advective)
        self.phase_seconds["integration"] += time.perf_counter() - t0
        dt = dt_adv
        if end_time is not None:
            dt = min(dt, end_time - self.time)
        if not overlapped:
            t0 = time.perf_counter()
            with self._kernel_event("skin_build"):
                self._lists_for_step(vmax, amax, dt)
            self.phase_seconds["cll"] += time.perf_counter() - t0
        self._last_step = (vmax, amax, dt)
        if self.shepard_every and self.step_count > 0 \
                and self.step_count % self.shepard_every == 0:
            t0 = time.perf_counter()
            self._call("sph_engine_shepard")
            self._host_same.discard("rho_scratch")
            self.phase_seconds["interactions"] += time.perf_counter() - t0
        nsub = max(1, int(math.ceil(dt / dt_ac)))
        dts = dt / nsub
        dtype = self.registry.dtype.type
        half = float(dtype(0.5 * dts))
        full = float(dtype(dts))
        t0 = time.perf_counter()
        E = ctypes.byref(d["E"])
        eager = self._eager_pull_ready()
        viewed = self._viewed
        if eager:
            self._copy_stream()
            marks = d["pull_events"]
            rc = L.sph_engine_substeps_marked(E, half, full, nsub,
                                              C_void(marks[0].cuda_event),
                                              C_void(marks[1].cuda_event), d["stream"])
            _native.check(rc, "engine_substeps_marked")
            self._deliver_tail()
            marks[2].record(d["tstream"])
            self._pull_overlapped(marks, marks[2])
        elif self.kernel_times is None:
            rc = L.sph_engine_substeps(E, half, full, nsub, d["stream"])
            _native.check(rc, "engine_substeps")
            self._deliver_tail()
        else:   # per-kernel CUDA-event timing (bench.py roofline pass)
            ms = (ctypes.c_float * 5)()
            rc = L.sph_engine_substeps_timed(E, half, full, nsub, ms, d["stream"])
            _native.check(rc, "engine_substeps_timed")
            self._deliver_tail()
            for k, name in enumerate(SUBSTEP_KERNELS):   # per sub-step average
                self.kernel_times.setdefault(name, []).append(ms[k] / nsub)
        self._call("sph_engine_stats", ctypes.c_int32(_native.STATS_NORMS))
        stats = self._read_stats()
        self.phase_seconds["interactions"] += time.perf_counter() - t0
        if self.kernel_times is not None:
            self._collect_events()
        self._view_streak = self._view_streak + 1 if viewed else 0
        self._viewed = False
        self.last_pull_overlapped = eager
        if eager:   # the host holds the step's result; the device stays authoritative
            d["cstream"].synchronize()
            self._host_stale = bool(stats.overflow)   # oflow changed: pull on view
        else:
            self._host_stale = True
        self.last_nsub = nsub
        self.last_nfix = int(stats.nfix)
        # list refreshes were rare: the next step checks and refreshes in one
        # pass (list_refresh "auto"); "pass" / "queue" force one of the paths
        if self.list_refresh == "auto":
            few = stats.nfix < 2e-4 * max(1, self.registry.particle_count) * nsub
        else:
            few = self.list_refresh == "pass"
        d["E"].few_refreshes = int(few)
        self._adapt_skin(stats.ndisp, nsub)
        if self._epoch is not None:   # largest path length since the epoch's build
            self._epoch["dmax"] = _bits_to_double(stats.dmax_bits)
            self._epoch["refresh"] = stats.ndisp / max(1, self.registry.particle_count * nsub)
        self.out_of_bounds += stats.oob + self._oob_walls
        self._finish_counts(stats, check=True)
        self.interaction_count += int(stats.interactions)
        self.step_count += 1
        self.time += dt
        c0 = float(self.registry.singular("c0"))
        # physics.py:554-564 with numpy's NaN-propagating min/max
        rho_min = (math.nan if stats.nan_flags & 1
                   else _key_to_double(stats.rho_min_key))
        if self.registry.particle_count and rho_min <= 0.0:
            raise SimulationUnstableError(
                f"non-positive density at step {self.step_count}")
        v2 = _key_to_double(stats.v2max_key) if self.registry.particle_count else 0.0
        if stats.nan_flags & 2:
            v2 = math.nan
        vmax_f = float(np.sqrt(self.registry.dtype.type(v2)))
        if self.registry.particle_count and vmax_f > 10.0 * c0:
            raise SimulationUnstableError(
                f"runaway velocity {vmax_f:.3g} at step {self.step_count}")
        return dt

    def snapshot_rows(self):
        """The snapshot fields (report.py:187-205) by original id as one
        (n, 2 dim + 2) run-dtype array: x[dim], v[dim], rho, p; row = id.
        Device-resident state: one gather kernel (sph_engine_snapshot) and
        one D2H copy into a reused pinned buffer; otherwise from the
        registry."""
        reg = self.registry
        n, d = reg.particle_count, reg.dim
        if self._dev is None or not self._host_stale:
            # the host arrays are current (read without a view: a view would
            # hand them to the caller and make the next step push)
            ids = reg.raw_view("id").astype(np.int64)
            out = np.empty((n, 2 * d + 2), reg.dtype)
            out[ids, :d] = reg.raw_view("x")
            out[ids, d:2 * d] = reg.raw_view("v")
            out[ids, 2 * d] = reg.raw_view("rho")
            out[ids, 2 * d + 1] = reg.raw_view("p")
            return out
        torch = torch_mod()
        dv = self._dev
        shape = (n, 2 * d + 2)
        if dv.get("snap") is None or tuple(dv["snap"].shape) != shape:
            dv["snap"] = torch.empty(shape, dtype=dv["tdtype"], device=dv["device"])
            dv["snap_host"] = torch.empty(shape, dtype=dv["tdtype"], pin_memory=True)
        with torch.cuda.stream(dv["tstream"]):
            rc = self._lib().sph_engine_snapshot(ctypes.byref(dv["E"]), ptr(dv["snap"]),
                                                 dv["stream"])
            _native.check(rc, "engine_snapshot")
            dv["snap_host"].copy_(dv["snap"], non_blocking=True)
        dv["tstream"].synchronize()
        return dv["snap_host"].numpy()

    def skin_entries(self):
        """(fluid, wall) totals of the current skin-list entry counts (the
        list bytes the sweeps stream; diagnostic)."""
        d = self._dev
        if d is None:
            return 0, 0
        E = d["E"]
        lc = d["T"]["lcount"]
        nf, nw = int(E.nf), int(E.n - E.nf)
        nf_pad = (nf + 31) // 32 * 32
        f = int(lc[:nf].sum().item()) if nf else 0
        w = int(lc[nf_pad:nf_pad + nw].sum().item()) if nw else 0
        return f, w

    def probe_candidates(self, location, reach, cap=1 << 16):
        """Fluid particles within (a conservatively widened) reach of a point,
        as registry-ordered host arrays (x, m, rho, p) in the run dtype, or
        None when there are more than cap of them."""
        torch = torch_mod()
        d = self._dev
        loc = np.zeros(3, np.float64)
        loc[:self.registry.dim] = np.asarray(location, np.float64)
        if "probe" not in d or d["probe"].shape[0] < cap * 7:
            d["probe"] = torch.empty(cap * 7, dtype=torch.float64, device=d["device"])
            d["probe_n"] = torch.zeros(1, dtype=torch.int32, device=d["device"])
        rc = self._lib().sph_engine_probe(
            ctypes.byref(d["E"]), loc.ctypes.data_as(ctypes.c_void_p),
            ctypes.c_double(reach * (1.0 + 1e-9) + 1e-300), ptr(d["probe"]), cap,
            ptr(d["probe_n"]), d["stream"])
        _native.check(rc, "engine_probe")
        k = int(d["probe_n"].item())
        if k > cap:
            return None
        rec = d["probe"][: 7 * k].view(k, 7).cpu().numpy()
        rec = rec[np.argsort(rec[:, 0], kind="stable")]
        dt = self.registry.dtype
        dim = self.registry.dim
        return (rec[:, 1:1 + dim].astype(dt), rec[:, 4].astype(dt), rec[:, 5].astype(dt),
                rec[:, 6].astype(dt))

    def _stability_check(self, c0):
        """physics.py:554-564 on the registry state."""
        rho = self.registry.view("rho")
        if rho.size and float(rho.min()) <= 0.0:
            raise SimulationUnstableError(
                f"non-positive density at step {self.step_count}")
        v = self.registry.view("v")
        if v.size:
            vmax = float(np.sqrt((v * v).sum(axis=1).max()))
            if vmax > 10.0 * c0:
                raise SimulationUnstableError(
                    f"runaway velocity {vmax:.3g} at step {self.step_count}")


# -- diagnostics (physics.py:569-606; host-side helpers) ----------------------

def total_energy(registry):
    m = registry.view("m")
    v = registry.view("v")
    x = registry.view("x")
    rho = registry.view("rho")
    wall = registry.view("wall")
    g = np.asarray(registry.singular("g"), dtype=np.float64)
    c0 = float(registry.singular("c0"))
    rho0 = float(registry.singular("rho0"))
    fluid = wall == 0
    ke = 0.5 * float((m[fluid] * (v[fluid] ** 2).sum(axis=1)).sum())
    pe = -float((m[fluid] * (x[fluid] @ g)).sum())
    dr = rho[fluid].astype(np.float64) - rho0
    ce = float((m[fluid] * c0 * c0 * dr * dr / (2.0 * rho0 * rho[fluid])).sum())
    return ke + pe + ce


def _shepard_probe(x, wall, m, rho, p, h, d, location):
    """physics.py:589-606 on arrays in registry order (the masked sums are
    numpy's, in that order)."""
    loc = np.asarray(location, dtype=np.float64)
    diff = x.astype(np.float64) - loc
    r = np.sqrt((diff * diff).sum(axis=1))
    mask = (r < 2.0 * h) & (wall == 0)
    if not mask.any():
        return 0.0
    w = np.array([kernel_W(ri, h, d) for ri in r[mask]])
    vol = (m[mask] / rho[mask]).astype(np.float64)
    den = float((w * vol).sum())
    if den == 0.0:
        return 0.0
    return float((p[mask] * w * vol).sum() / den)


def sample_pressure(registry, location):
    """Shepard-interpolated fluid pressure at a point (physics.py:589-606).

    While a device engine holds the state, only the fluid particles near the
    probe are fetched (sph_engine_probe) -- in registry order, so the
    reference's computation on them gives the same bits -- instead of pulling
    every field to the host."""
    h = float(registry.singular("h"))
    d = registry.dim
    eng = getattr(registry, "_engine", None)
    if eng is not None and getattr(eng, "_host_stale", False):
        sub = eng.probe_candidates(location, 2.0 * h)
        if sub is not None:
            x, m, rho, p = sub
            return _shepard_probe(x, np.zeros(len(m), np.uint32), m, rho, p, h, d, location)
    return _shepard_probe(registry.view("x"), registry.view("wall"), registry.view("m"),
                          registry.view("rho"), registry.view("p"), h, d, location)

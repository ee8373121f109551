"""ctypes binding of libsphb200.so (include/sph_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

c_void_p = C.c_void_p
c_i64 = C.c_int64
c_i32 = C.c_int32
c_f32 = C.c_float
c_f64 = C.c_double
c_size = C.c_size_t

SPH_OK = 0
SPH_ERR_INVALID = 1
SPH_ERR_CUDA = 2
SPH_ERR_NEGATIVE_KEY = 3
SPH_ERR_WORKSPACE = 4
SPH_ERR_UNSUPPORTED = 5
NEIGHBOR_CAPACITY = 256


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available."""


class NativeError(RuntimeError):
    pass


def _sweep_fields(real):
    P = c_void_p
    return [
        ("x", P), ("v", P), ("rho", P), ("p", P), ("m", P),
        ("wall", P), ("ids", P), ("offsets", P), ("pids", P),
        ("drho", P), ("dvdt", P), ("nnb", P), ("oflow", P), ("rho_new", P),
        ("g", real * 3), ("origin", real * 3), ("shape", c_i64 * 3),
        ("cell_size", real), ("cutoff", real), ("h", real), ("alpha_d", real),
        ("c0", real), ("rho0", real), ("alpha_visc", real), ("eps_h2", real),
        ("n", c_i64), ("dim", c_i32), ("reserved", c_i32),
    ]


class SphSweepArgs_f32(C.Structure):
    _fields_ = _sweep_fields(c_f32)


class SphSweepArgs_f64(C.Structure):
    _fields_ = _sweep_fields(c_f64)


class SphHaloPlan(C.Structure):
    MAX_PEERS = 8
    _fields_ = [
        ("npeers", c_i32), ("peer", c_i32 * 8),
        ("send_phys", C.c_void_p * 2), ("recv_phys", C.c_void_p * 2),
        ("send_off", (C.c_int64 * 9) * 2), ("recv_off", (C.c_int64 * 9) * 2),
        ("send_buf", C.c_void_p), ("recv_buf", C.c_void_p),
    ]


class SphStepStats(C.Structure):
    _fields_ = [
        ("vmax_bits", C.c_uint64), ("amax_bits", C.c_uint64),
        ("interactions", C.c_uint64), ("rho_min_key", C.c_uint64),
        ("v2max_key", C.c_uint64), ("dmax_bits", C.c_uint64),
        ("overflow", C.c_uint32), ("oob", C.c_uint32),
        ("oob_walls", C.c_uint32), ("nfix", C.c_uint32),
        ("nan_flags", C.c_uint32), ("push_error", C.c_uint32),
        ("fluid_seen", C.c_uint32), ("ndisp", C.c_uint32),
    ]


class SphEngine(C.Structure):
    P = c_void_p
    _fields_ = [
        ("n", c_i64), ("nf", c_i64), ("ncells", c_i64),
        ("dim", c_i32), ("key_bits", c_i32),
        ("pos", P * 2), ("vel", P * 2), ("rp", P * 2), ("rq", P), ("dvdt", P), ("drho", P),
        ("id", P), ("nnb", P), ("refpos", P),
        ("rho_scratch_id", P), ("oflow_id", P), ("wall_id", P), ("vol_id", P),
        ("owned_id", P),
        ("offs_f", P), ("offs_w", P),
        ("lists", P), ("lcount", P), ("acount", P), ("nww", P), ("elist", P),
        ("cell0", P), ("disp", P), ("queue", P), ("qcount", P),
        ("ws", P), ("ws_bytes", c_size),
        ("stats", P),
        ("g", c_f64 * 3), ("origin", c_f64 * 3), ("shape", c_i64 * 3),
        ("cell_size", c_f64), ("cutoff", c_f64), ("h", c_f64), ("alpha_d", c_f64),
        ("c0", c_f64), ("rho0", c_f64), ("alpha_visc", c_f64), ("eps_h2", c_f64),
        ("skin", c_f64),
        ("cur_v", c_i32), ("cur_rp", c_i32), ("cur_pos", c_i32), ("drifted", c_i32), ("f64", c_i32), ("lists_ready", c_i32),
        ("period", c_f64 * 3),
        ("disp0", P),
        ("few_refreshes", c_i32), ("nww_ready", c_i32),
        ("id_range", c_i64),
        ("key_sorted", P), ("key_prev", P), ("perm", P), ("inv", P),
        ("lists_alt", P), ("lcount_alt", P),
        ("lists_stale", c_i32), ("cll_fresh", c_i32),
        ("cellmax", P), ("blockmax", P),
    ]


class SphRows(C.Structure):
    _fields_ = [("f", c_void_p * 13)]


SPH_MAX_RANKS = 64


class SphSlabGeom(C.Structure):
    _fields_ = [
        ("nplanes", c_i64), ("origin", c_f64 * 3), ("cell_size", c_f64),
        ("shape", c_i64 * 3),
        ("nranks", c_i32), ("rank", c_i32), ("periodic", c_i32), ("halo", c_i32),
        ("cuts", c_i64 * (SPH_MAX_RANKS + 1)),
        ("npeers", c_i32), ("peer", c_i32 * 8),
    ]


ABI_VERSION = 16   # include/sph_b200.h SPH_ABI_VERSION (SphEngine layout)
STATS_RESET = 1
STATS_NORMS = 2
# sph_engine_phase / halo records (include/sph_b200.h)
PHASE_KICK_DRIFT, PHASE_CONTINUITY, PHASE_WALL, PHASE_MOMENTUM = 0, 1, 2, 3
PHASE_INIT_WALL, PHASE_INIT_MOMENTUM, PHASE_MOMENTUM_NEXT = 4, 5, 6
HALO_XV, HALO_RP_NEXT, HALO_RP_CUR = 0, 1, 2
LATTICE_ALL, LATTICE_TANK, LATTICE_NOT_IN = 0, 1, 2

# name -> (restype, argtypes)
_P = c_void_p
_PROTOS = {
    "sph_abi_version": (c_i32, []),
    "sph_last_error": (C.c_char_p, []),
    "sph_kernel_launches": (C.c_longlong, []),
    "sph_sweep_workspace_bytes": (c_size, [c_i64]),
    "sph_cll_workspace_bytes": (c_size, [c_i64, c_i64]),
    "sph_sort_workspace_bytes": (c_size, [c_i64]),
    "sph_engine_workspace_bytes": (c_size, [c_i64, c_i64, c_i32]),
    "sph_engine_workspace_bytes_ids": (c_size, [c_i64, c_i64, c_i32, c_i64]),
    "sph_radix_sort_perm": (c_i32, [_P, c_i64, _P, _P, c_size, _P]),
    "sph_gather": (c_i32, [_P, _P, _P, c_i64, c_i32, _P]),
    "sph_copy": (c_i32, [_P, _P, c_i64, _P]),
    "sph_selftest_div": (c_i32, [c_f64, c_i64, C.c_uint64, _P, _P]),
    "sph_selftest_pair_fac": (c_i32, [c_f64, c_f64, C.c_uint32, C.c_uint32, _P, _P, _P]),
    "sph_selftest_round_f32": (c_i32, [c_i64, C.c_uint64, _P, _P, _P]),
    "sph_engine_push": (c_i32, [_P] * 14 + [_P]),
    "sph_engine_push_begin": (c_i32, [_P] * 4 + [_P]),
    "sph_engine_push_end": (c_i32, [_P] * 11 + [_P]),
    "sph_engine_push_tail": (c_i32, [_P] * 5 + [_P]),
    "sph_engine_pull": (c_i32, [_P] * 14 + [_P]),
    "sph_engine_pull_fields": (c_i32, [_P, C.c_uint32] + [_P] * 13 + [_P]),
    "sph_engine_rebuild_cll": (c_i32, [_P, _P]),
    "sph_engine_ref_sort": (c_i32, [_P, _P]),
    "sph_engine_initialize": (c_i32, [_P, _P]),
    "sph_engine_build_lists": (c_i32, [_P, c_f64, _P]),
    "sph_engine_shepard": (c_i32, [_P, _P]),
    "sph_engine_substep": (c_i32, [_P, c_f64, c_f64, _P]),
    "sph_engine_substep_timed": (c_i32, [_P, c_f64, c_f64, _P, _P]),
    "sph_engine_stats": (c_i32, [_P, c_i32, _P]),
    "sph_engine_substeps": (c_i32, [_P, c_f64, c_f64, c_i32, _P]),
    "sph_engine_substeps_timed": (c_i32, [_P, c_f64, c_f64, c_i32, _P, _P]),
    "sph_engine_substeps_marked": (c_i32, [_P, c_f64, c_f64, c_i32, _P, _P, _P]),
    "sph_engine_phase": (c_i32, [_P, c_i32, c_f64, c_f64, _P]),
    "sph_engine_probe": (c_i32, [_P, _P, c_f64, _P, c_i32, _P, _P]),
    "sph_engine_snapshot": (c_i32, [_P, _P, _P]),
    "sph_engine_maintain_lists": (c_i32, [_P, _P]),
    "sph_slab_record_words": (c_i32, [c_i32, c_i32]),
    "sph_stats_allreduce": (c_i32, [_P, _P, c_i32, _P]),
    "sph_slab_classify": (c_i32, [_P, _P, _P, c_i64, c_i32, c_i32, _P, _P, _P]),
    "sph_slab_pack": (c_i32, [_P, c_i32, c_i32, _P, c_i64, _P, _P]),
    "sph_slab_unpack": (c_i32, [_P, c_i64, _P, c_i32, c_i32, c_i64, _P]),
    "sph_slab_gather": (c_i32, [_P, _P, c_i64, _P, c_i32, c_i32, c_i64, _P]),
    "sph_engine_halo_width": (c_i32, [c_i32]),
    "sph_engine_pack": (c_i32, [_P, c_i32, _P, c_i64, _P, _P]),
    "sph_halo_pack": (c_i32, [_P, _P, c_i32, c_i32, _P]),
    "sph_halo_unpack": (c_i32, [_P, _P, c_i32, c_i32, _P]),
    "sph_comm_id_bytes": (c_size, []),
    "sph_comm_unique_id": (c_i32, [_P]),
    "sph_comm_init": (c_i32, [_P, c_i32, c_i32, _P]),
    "sph_comm_destroy": (c_i32, [_P]),
    "sph_halo_exchange": (c_i32, [_P, _P, _P, c_i32, c_i32, _P]),
    "sph_engine_substeps_slab": (c_i32, [_P, _P, _P, c_f64, c_f64, c_i32, _P]),
    "sph_engine_unpack": (c_i32, [_P, c_i32, _P, c_i64, _P, _P]),
    "sph_lattice_workspace_bytes": (c_size, [c_i32, _P, _P]),
    "sph_lattice_points": (c_i32, [c_i32, _P, _P, c_f64, _P, c_i32, _P, _P, _P, _P,
                                   _P, _P, _P, c_size, _P]),
}
for _sfx, _real in (("f32", c_f32), ("f64", c_f64)):
    for _k in ("continuity", "momentum", "wall_pressure", "density_summation",
               "shepard"):
        _PROTOS[f"sph_{_k}_{_sfx}"] = (c_i32, [_P, _P, c_size, _P])
    _PROTOS[f"sph_neighbors_{_sfx}"] = (c_i32, [_P, c_i64, c_i64, _P, _P, _P])
    _PROTOS[f"sph_kick_{_sfx}"] = (c_i32, [_P, _P, _P, c_i64, c_i32, _real, _P])
    _PROTOS[f"sph_drift_{_sfx}"] = (c_i32, [_P, _P, _P, c_i64, c_i32, _real, _P])
    _PROTOS[f"sph_density_update_{_sfx}"] = (
        c_i32, [_P, _P, _P, _P, c_i64, _real, _real, _real, _P])
    _PROTOS[f"sph_vmax_{_sfx}"] = (c_i32, [_P, c_i64, c_i32, _P, _P])
    _PROTOS[f"sph_cell_keys_{_sfx}"] = (
        c_i32, [_P, c_i64, c_i32, _P, _real, _P, _P, _P, _P])
    _PROTOS[f"sph_cll_build_{_sfx}"] = (
        c_i32, [_P, c_i64, c_i32, _P, _real, _P, _P, _P, _P, _P, c_size, _P])

EXPORTED = tuple(sorted(_PROTOS))

_LIB = None
_LIB_PERIODIC = None


def library_path(periodic=False):
    """The in-tree library; SPH_B200_LIB overrides it (A/B variant builds).
    periodic: the periodic-box build (libsphb200_periodic.so)."""
    if periodic:
        return os.environ.get("SPH_B200_LIB_PERIODIC") or _build.LIB_PERIODIC
    return os.environ.get("SPH_B200_LIB") or _build.LIB


def load(path=None, periodic=False):
    """Load the shared library and declare prototypes (no GPU needed)."""
    global _LIB, _LIB_PERIODIC
    if path is None:
        cached = _LIB_PERIODIC if periodic else _LIB
        if cached is not None:
            return cached
    p = path or library_path(periodic)
    if not os.path.exists(p):
        raise NativeUnavailable(
            f"{p} is missing: run `python -m paper_2603_11868_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(p)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sph_abi_version() != ABI_VERSION:
        raise NativeUnavailable("libsphb200.so ABI version mismatch")
    if path is None:
        if periodic:
            _LIB_PERIODIC = lib
        else:
            _LIB = lib
    return lib


def lib(periodic=False):
    return load(periodic=periodic)


def last_error():
    """The last error message of the loaded libraries (bounded, periodic)."""
    msgs = []
    for L in (_LIB, _LIB_PERIODIC):
        if L is not None:
            m = L.sph_last_error()
            if m:
                msgs.append(m.decode())
    return "; ".join(msgs)


def check(rc, what):
    """Map an SPH_ERR_* status to the reference's exception classes."""
    if rc == SPH_OK:
        return
    detail = last_error()
    if rc == SPH_ERR_NEGATIVE_KEY:
        raise ValueError("radix sort keys must be non-negative")
    if rc == SPH_ERR_INVALID:
        raise TypeError(f"{what}: invalid arguments ({detail})")
    if rc == SPH_ERR_UNSUPPORTED:
        raise ValueError(f"{what}: unsupported size ({detail})")
    raise NativeError(f"{what} failed with status {rc}: {detail}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    load()


def sweep_struct(dtype):
    return SphSweepArgs_f32 if np.dtype(dtype) == np.float32 else SphSweepArgs_f64


def sfx(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"unsupported precision {dt}")

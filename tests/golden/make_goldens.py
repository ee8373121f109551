"""Generate the golden fixtures in this directory from the REFERENCE package.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_goldens.py

It imports ``minisph`` (reference ``pkg/src/minisph``) read-only and writes
small ``.npz`` fixtures next to this script.  Nothing at test or bench time
reads ``/root/reference``; only these committed outputs travel.

Fixtures
--------
``traj_<case>_<prec>.npz``
    A whole-step trajectory through the reference ``Simulation``
    (physics.py:416-564): per step ``dt`` (advance's return value), ``nsub``
    (recomputed with compute_timestep, physics.py:386-400 / 512-516, which is
    pure and reads only v and dvdt), the cumulative interaction count, the
    out-of-bounds count, and a SHA-256 per discrete variable of the field
    ordered BY ID and of the field in the registry's PHYSICAL order.  Full
    by-id arrays are kept at a few ``full_steps`` (0 == after initialize()).
``kat_kernels_<prec>.npz``
    Single-sweep known answers on the reference's own test clouds
    (tests/test_physics.py:54-66 noisy cloud, with walls added): continuity,
    momentum, wall pressure, density summation, Shepard, kick/drift/density
    update, VMAX reductions, plus the cell linked list and ordered neighbour
    visits of sampled particles.
``kat_sort.npz``
    Radix / stable sort permutations on the rng(7) key sets of
    tests/test_acceptance.py:76-89 (subset) and tests/test_sorting.py:17-20.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import minisph  # noqa: E402  (reference, imported read-only)
from minisph import physics as P  # noqa: E402
from minisph.cases import CaseConfig, load_config  # noqa: E402
from minisph.execution import ExecutionPolicy, particle_for, particle_reduce  # noqa: E402
from minisph.neighborhood import (UniformGrid, build_cell_linked_list,  # noqa: E402
                                  collect_neighbors, compute_cell_keys,
                                  NEIGHBOR_CAPACITY)
from minisph.report import build_case  # noqa: E402
from minisph.sorting import (comparison_sort_permutation,  # noqa: E402
                             radix_sort_permutation)

PAR = ExecutionPolicy.parallel(os.cpu_count() or 1)
FIELDS = ("x", "v", "rho", "p", "m", "Vol", "drho", "dvdt", "rho_scratch",
          "id", "wall", "nnb", "oflow")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def by_id(reg, name):
    order = np.argsort(reg.view("id"), kind="stable")
    return reg.view(name)[order]


def kleefsman_cfg(dp, precision):
    path = os.path.join(os.path.dirname(minisph.__file__), "data",
                        "kleefsman.cfg")
    cfg = load_config(path)
    cfg.dp = dp
    cfg.precision = precision
    return cfg


def trajectory(tag, cfg, steps, full_steps, sort_every=100,
               shepard_every=200):
    reg, grid = build_case(cfg)
    sim = P.Simulation(reg, grid, PAR, dt_max=cfg.dt_max,
                       sort_every=sort_every, shepard_every=shepard_every)
    out = {"n": reg.particle_count, "dim": reg.dim,
           "grid_origin": np.asarray(grid.origin, np.float64),
           "grid_shape": np.asarray(grid.shape, np.int64),
           "grid_cell_size": np.float64(grid.cell_size)}
    # initial (pre-initialize) state, by id == physical at this point
    for f in FIELDS:
        out[f"init_{f}"] = reg.view(f).copy()
    for s in ("rho0", "c0", "h", "dp", "alpha_visc", "g"):
        out[f"sing_{s}"] = np.asarray(reg.singular(s))
    sim.initialize()
    rec_dt, rec_nsub, rec_ic, rec_oob, rec_time = [], [], [], [], []
    hashes_id = {f: [] for f in FIELDS}
    hashes_phys = {f: [] for f in FIELDS}

    def record(step):
        for f in FIELDS:
            hashes_id[f].append(sha(by_id(reg, f)))
            hashes_phys[f].append(sha(reg.view(f)))
        if step in full_steps:
            for f in FIELDS:
                out[f"s{step}_{f}"] = by_id(reg, f).copy()

    record(0)
    rec_dt.append(0.0); rec_nsub.append(0)
    rec_ic.append(sim.interaction_count); rec_oob.append(sim.out_of_bounds)
    rec_time.append(sim.time)
    for step in range(1, steps + 1):
        dt_ac, dt_adv = P.compute_timestep(PAR, reg, sim.dt_max)
        nsub = max(1, int(math.ceil(dt_adv / dt_ac)))
        dt = sim.advance()
        assert dt == dt_adv
        rec_dt.append(dt); rec_nsub.append(nsub)
        rec_ic.append(sim.interaction_count); rec_oob.append(sim.out_of_bounds)
        rec_time.append(sim.time)
        record(step)
    out["dt"] = np.asarray(rec_dt, np.float64)
    out["nsub"] = np.asarray(rec_nsub, np.int64)
    out["interactions"] = np.asarray(rec_ic, np.int64)
    out["out_of_bounds"] = np.asarray(rec_oob, np.int64)
    out["time"] = np.asarray(rec_time, np.float64)
    for f in FIELDS:
        out[f"hid_{f}"] = np.asarray(hashes_id[f])
        out[f"hph_{f}"] = np.asarray(hashes_phys[f])
    out["full_steps"] = np.asarray(sorted(full_steps), np.int64)
    path = os.path.join(HERE, f"traj_{tag}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: N={reg.particle_count} steps={steps} "
          f"nsub={sorted(set(rec_nsub[1:]))}")


def noisy_cloud_with_walls(dtype, seed=7, n=400, dp=0.02, dim=2):
    """tests/test_physics.py:54-66 noisy cloud (+ a wall strip, + 3D)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from _support import make_cloud_registry, grid_around, lattice_positions
    rng = np.random.default_rng(seed)
    if dim == 2:
        side = int(round(math.sqrt(n)))
        pos = lattice_positions((side, side), dp)
        g = (0.0, -9.81)
    else:
        side = int(round(n ** (1 / 3)))
        pos = lattice_positions((side, side, side), dp)
        g = (0.0, 0.0, -9.81)
    pos += rng.normal(0.0, 0.05 * dp, pos.shape)
    reg = make_cloud_registry(pos, dp=dp, dtype=dtype, gravity=g)
    reg.view("v")[:] = rng.normal(0.0, 0.1, pos.shape)
    rho = 1000.0 * (1.0 + rng.normal(0.0, 1e-3, pos.shape[0]))
    reg.view("rho")[:] = rho
    reg.view("p")[:] = P.eos_pressure(rho, 1000.0, 20.0)
    reg.view("dvdt")[:] = rng.normal(0.0, 5.0, pos.shape)
    reg.view("drho")[:] = rng.normal(0.0, 1.0, pos.shape[0])
    # bottom layers become walls (exercises the wall branches)
    low = pos[:, -1] < 3 * dp
    reg.view("wall")[low] = 1
    # shuffle the physical order so within-cell order != id order
    perm = np.random.default_rng(seed + 1).permutation(reg.particle_count)
    reg.apply_permutation(perm)
    cutoff = 2.0 * float(reg.singular("h"))
    grid = grid_around(reg.view("x").astype(np.float64), cutoff, pad=0.0)
    return reg, grid


def kat_kernels(prec):
    dtype = np.float32 if prec == "f32" else np.float64
    out = {}
    for dim in (2, 3):
        reg, grid = noisy_cloud_with_walls(dtype, dim=dim,
                                           n=400 if dim == 2 else 512)
        cll = build_cell_linked_list(PAR, reg.view("x"), grid)
        pre = f"d{dim}_"
        for f in FIELDS:
            out[pre + "in_" + f] = reg.view(f).copy()
        out[pre + "grid_origin"] = np.asarray(grid.origin, np.float64)
        out[pre + "grid_shape"] = np.asarray(grid.shape, np.int64)
        out[pre + "grid_cell_size"] = np.float64(grid.cell_size)
        for s in ("rho0", "c0", "h", "dp", "alpha_visc", "g"):
            out[pre + "sing_" + s] = np.asarray(reg.singular(s))
        out[pre + "cll_offsets"] = cll.offsets.copy()
        out[pre + "cll_pids"] = cll.particle_ids.copy()
        keys, oob = compute_cell_keys(reg.view("x"), grid)
        out[pre + "keys"] = keys
        fa = P.force_args(reg, cll)
        out[pre + "force_scalars"] = np.asarray(fa[16:], dtype)
        # ordered neighbour lists (physical j) of every particle
        nbr = np.full((reg.particle_count, NEIGHBOR_CAPACITY), -1, np.int64)
        cnts = np.zeros(reg.particle_count, np.int64)
        buf = np.empty(NEIGHBOR_CAPACITY, np.int64)
        for i in range(reg.particle_count):
            c = collect_neighbors(i, fa[0], fa[6], fa[8], fa[9], fa[10],
                                  fa[16], fa[11], fa[17], buf)
            cnts[i] = c
            nbr[i, :c] = buf[:c] & 0xFFFFFFFF
        out[pre + "nbr_count"] = cnts
        out[pre + "nbr_list"] = nbr[:, :max(1, cnts.max())]
        # sweeps, each from the same input state
        state = {f: reg.view(f).copy() for f in FIELDS}

        def reset():
            for f in FIELDS:
                reg.view(f)[:] = state[f]

        P.evaluate_continuity(PAR, reg, cll)
        out[pre + "cont_drho"] = reg.view("drho").copy()
        reset()
        P.evaluate_momentum(PAR, reg, cll)
        out[pre + "mom_dvdt"] = reg.view("dvdt").copy()
        out[pre + "mom_nnb"] = reg.view("nnb").copy()
        reset()
        P.extrapolate_wall_pressure(PAR, reg, cll)
        out[pre + "wp_p"] = reg.view("p").copy()
        out[pre + "wp_rho"] = reg.view("rho").copy()
        out[pre + "wp_nnb"] = reg.view("nnb").copy()
        reset()
        minisph.dispatch_dynamics(PAR, P.DensitySummationDynamics(reg, cll))
        out[pre + "ds_rho"] = reg.view("rho").copy()
        reset()
        h = reg.singular("h")
        dt = reg.dtype.type
        args = (reg.view("x"), reg.view("rho"), reg.view("m"),
                reg.view("wall"), reg.view("id"), cll.offsets,
                cll.particle_ids, cll.grid.origin.astype(reg.dtype),
                cll.grid.shape_array(), reg.view("rho_scratch"),
                dt(cll.grid.cell_size), dt(2.0 * h), dt(h),
                dt(P.wendland_alpha(h, reg.dim)))
        particle_for(PAR, reg.particle_count, P.SHEPARD, args)
        out[pre + "shep_rho_new"] = reg.view("rho_scratch").copy()
        reset()
        half = dt(0.5 * 1.2345e-4)
        full = dt(1.2345e-4)
        particle_for(PAR, reg.particle_count, P.KICK,
                     (reg.view("v"), reg.view("dvdt"), reg.view("wall"), half))
        out[pre + "kick_v"] = reg.view("v").copy()
        particle_for(PAR, reg.particle_count, P.DRIFT,
                     (reg.view("x"), reg.view("v"), reg.view("wall"), full))
        out[pre + "drift_x"] = reg.view("x").copy()
        particle_for(PAR, reg.particle_count, P.DENSITY_UPDATE,
                     (reg.view("rho"), reg.view("p"), reg.view("drho"),
                      reg.view("wall"), full, dt(reg.singular("c0")),
                      dt(reg.singular("rho0"))))
        out[pre + "du_rho"] = reg.view("rho").copy()
        out[pre + "du_p"] = reg.view("p").copy()
        out[pre + "du_scalars"] = np.asarray([half, full], dtype)
        reset()
        out[pre + "vmax"] = np.float64(particle_reduce(
            PAR, reg.particle_count, P.VMAX_SPEC, (reg.view("v"),)))
        out[pre + "amax"] = np.float64(particle_reduce(
            PAR, reg.particle_count, P.VMAX_SPEC, (reg.view("dvdt"),)))
        out[pre + "timestep"] = np.asarray(P.compute_timestep(PAR, reg, 1e-3))
    path = os.path.join(HERE, f"kat_kernels_{prec}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


def kat_sort():
    out = {}
    rng = np.random.default_rng(7)
    pol = ExecutionPolicy.parallel_device(8)
    sets = []
    for _ in range(40):
        n = int(10 ** rng.uniform(0.0, 5.0))
        keys = rng.integers(0, int(rng.choice([16, 2**16, 2**40])), size=n)
        sets.append(keys)
    # keys are regenerated from rng(7) by the tests; only hashes are kept
    kh, ph = [], []
    for k, keys in enumerate(sets):
        perm = radix_sort_permutation(pol, keys)
        assert np.array_equal(perm, comparison_sort_permutation(keys))
        kh.append(sha(keys.astype(np.int64)))
        ph.append(sha(perm.astype(np.int64)))
    out["keys_sha"] = np.asarray(kh)
    out["perm_sha"] = np.asarray(ph)
    out["nsets"] = np.int64(len(sets))
    out["kat_keys"] = np.array([3, 1, 3, 1, 2, 1], np.int64)
    out["kat_perm"] = comparison_sort_permutation(out["kat_keys"])
    path = os.path.join(HERE, "kat_sort.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


def main():
    which = set(sys.argv[1:]) or {"kat", "sort", "traj2d", "traj3d"}
    if "sort" in which:
        kat_sort()
    if "kat" in which:
        kat_kernels("f32")
        kat_kernels("f64")
    if "traj2d" in which:
        trajectory("dambreak2d_f32",
                   CaseConfig(case="dambreak2d", dp=0.025, precision="f32"),
                   steps=210, full_steps={0, 1, 2, 5, 100, 101, 201})
        trajectory("dambreak2d_f64",
                   CaseConfig(case="dambreak2d", dp=0.025, precision="f64"),
                   steps=30, full_steps={0, 1})
        # coarse 2D run long enough for the flow to develop (cell crossings,
        # advective-CFL-limited steps, several sort/Shepard passes)
        trajectory("dambreak2d_coarse_f32",
                   CaseConfig(case="dambreak2d", dp=0.05, precision="f32"),
                   steps=700, full_steps={0, 700})
    if "traj3d" in which:
        trajectory("kleefsman3d_f32", kleefsman_cfg(0.04, "f32"),
                   steps=205, full_steps={0, 1})


if __name__ == "__main__":
    main()

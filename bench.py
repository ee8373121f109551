"""Benchmark: full-time-step particle-updates/s of the WCSPH dam break on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2d1m|3d4m|3d16m|2dref]
    python bench.py --impl reference ...      (CPU reference arm)

One "step" = one Simulation.advance (physics.py:489-552): CLL rebuild, the
time-step reductions and nsub acoustic sub-steps, exactly the reference's
work.  value = particles x steps / device time (CUDA events, summed over
steps; L2 flushed between steps; max over ranks).  At N > 1 the same
configuration is slab-partitioned over the N GPUs (distributed.py: balanced
axis-0 slabs, 2-plane halos, NCCL halo exchange and migration; strong
scaling, results bit-identical to one GPU).

Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (description, builder kwargs)
    "2dref": ("config 1: reference 2D dam break, dp=0.025 (N=5,153)",
              dict(kind="2d", dp=0.025)),
    "2d1m": ("config 2: 2D dam break at 1M particles, dp=0.00144 (N=997,518)",
             dict(kind="2d", dp=0.00144)),
    "3d4m": ("config 3: 3D Kleefsman dam break at 4M, dp=0.00608 (N=3,988,296)",
             dict(kind="3d", dp=0.00608)),
    "3d16m": ("config 4: 3D Kleefsman dam break at 16M, dp=0.00371 (N=16,005,253)",
              dict(kind="3d", dp=0.00371)),
    # config 5's per-GPU share (64M on 8 GPUs): not constructible in the
    # reference (no periodic boundaries); SURVEY.md 8f f4
    "tg8m": ("config 5 per GPU: 3D periodic Taylor-Green vortex, 200^3 = 8M particles "
             "(libsphb200_periodic.so; beyond the reference, parity vs the oracle's "
             "periodic restatement)", dict(kind="tg", n=200)),
}
METRIC = "particle-updates/sec (full time step)"
UNIT = "particle-updates/s"
SUBSTEP_KERNELS = ("kick_drift", "list_filter", "continuity_du", "wall_pressure",
                   "momentum_kick")


_OUT_FD = None


def emit(line):
    """The one JSON line on the process's original stdout (NCCL and other
    libraries may print banners on fd 1; those are diverted to stderr)."""
    data = (json.dumps(line) + "\n").encode()
    if _OUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_OUT_FD, data)


def tg_side(name, world=1):
    """Weak scaling of config 5: n^3 = world x 200^3 particles (8 GPUs: 400^3
    = 64M, BASELINE config 5)."""
    return int(round(CONFIGS[name][1]["n"] * world ** (1.0 / 3.0)))


def case_config(name, world=1):
    from paper_2603_11868_b200 import cases
    spec = CONFIGS[name][1]
    if spec["kind"] == "tg":
        return cases.taylor_green_config(3, tg_side(name, world), precision="f32")
    if spec["kind"] == "2d":
        return cases.CaseConfig(case="dambreak2d", dp=spec["dp"], precision="f32")
    return cases.kleefsman_config(dp=spec["dp"], precision="f32")


def build_case(name, world=1):
    """Host placement (the reference's numpy lattice restated): the CPU arms
    and the slab path start from it."""
    from paper_2603_11868_b200 import cases
    return cases.build_case(case_config(name, world))


def data_label(name):
    if CONFIGS[name][1]["kind"] == "tg":
        return "synthetic (periodic Taylor-Green lattice, analytic initial field)"
    return "synthetic (reference lattice dam break, deterministic)"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# -- algorithmic bytes -----------------------------

def kernel_bytes(name, d, nf, nw, nnb_f, nnb_w, nnb_wf):
    """Compulsory DRAM bytes of one launch: each field the kernel must read
    once, each field it must write once (fp32 run, uint32 index); gathered
    neighbour data is assumed cache-resident (SURVEY.md section 8d model)."""
    if name == "kick_drift":       # read x v a, write x v (first sub-step only)
        return nf * 20 * d
    if name == "list_filter":      # k_mark: read cell0, disp (fix-ups extra)
        return (nf + nw) * 8
    if name == "continuity_du":    # read x v rho m + list, write drho rho p
        return nf * (8 * d + 8 + 4 + 12) + 4 * nnb_f
    if name == "wall_pressure":    # read x + list, write rho p nnb drho
        return nw * (4 * d + 4 + 16) + 4 * nnb_wf
    if name == "momentum_kick":    # read x v rho p m + list, write dvdt v x
        return nf * (20 * d + 20) + 4 * nnb_f
    raise KeyError(name)


def step_bytes_model(d, n, nf, nw, nsub, ncells, passes):
    """B_full = nsub*B_sub + B_step per particle-update."""
    w = nw / n
    b_sub = 28 * d + 44 + w * (4 * d + 16)
    b_step = 24 * d + 8 + 16 * passes + 4 + 8 * ncells / n
    return nsub * b_sub + b_step


# -- clocks ---------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        """Spawn the sampler (20 ms period) and wait for its first row, so the
        timed region that follows is covered from its start."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        deadline = time.perf_counter() + 5.0
        while not self.rows and time.perf_counter() < deadline:
            time.sleep(0.005)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [c.strip() for c in line.split(",")]))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=5)
        # samples read within the timed region (one period of slack after it)
        rows = list(self.rows)
        if self.t0 is not None:
            t1 = (self.t1 or time.perf_counter()) + 0.025
            rows = [r for r in rows if self.t0 <= r[0] <= t1]
        self.rows = [r[1] for r in rows]
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(r) > 2 + k and r[2 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# -- CPU arms -------------------------------------------------------------------

def cpu_oracle_run(name, steps, budget_s, warmup=0, world=1):
    """Time the oracle port (all host threads) on the same configuration:
    initialize() and ``warmup`` steps untimed (bounded by budget_s / 2), then
    up to ``steps`` advective steps bounded by ``budget_s`` seconds.
    Returns (PU/s, steps_done, seconds, threads, nsubs)."""
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    from oracle.oracle import OracleSim
    reg, grid = build_case(name, world if CONFIGS[name][1]["kind"] == "tg" else 1)
    sim = OracleSim.from_registry(reg, grid)
    sim.initialize()
    t0 = time.perf_counter()
    for _ in range(warmup):
        sim.advance()
        if time.perf_counter() - t0 > budget_s / 2:
            break
    n = reg.particle_count
    done, total = 0, 0.0
    nsubs = []
    while done < steps:
        t0 = time.perf_counter()
        sim.advance()
        total += time.perf_counter() - t0
        done += 1
        nsubs.append(sim.last_nsub)
        if total >= budget_s:
            break
    return n * done / total, done, total, int(os.environ["OMP_NUM_THREADS"]), nsubs


def reference_arm(args, rank, world):
    if rank != 0:
        return
    pus, done, secs, thr, nsubs = cpu_oracle_run(args.config, max(1, args.steps),
                                                 budget_s=args.cpu_budget,
                                                 warmup=args.warmup, world=world)
    line = {
        "impl": "reference", "metric": METRIC, "value": pus, "unit": UNIT,
        "n_gpus": world, "steps": done, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / done, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (mixed f64)",
        "data": data_label(args.config),
        "config": {"workload": CONFIGS[args.config][0], "case": args.config},
        "cpu_baseline": {
            "value": pus, "unit": UNIT, "cores": thr, "kind": "port",
            "sample": f"{done} full advective step(s) (nsub={nsubs}) after an "
                      f"untimed initialize() + up to {args.warmup} warm-up steps, "
                      f"C port of the reference "
                      f"(oracle/sph_oracle.c, bit-identical), OpenMP {thr} threads"},
        "e2e": {"value": pus, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


# -- GPU arm --------------------------------------------------------------------

def gpu_arm(args, rank, world, local_rank):
    import numpy as np
    import torch
    from paper_2603_11868_b200 import ExecutionPolicy, _native
    from paper_2603_11868_b200.physics import Simulation

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2603_11868_b200.physics import grid_is_periodic
    from paper_2603_11868_b200 import cases
    cfg = case_config(args.config)
    t_setup = time.perf_counter()
    if CONFIGS[args.config][1]["kind"] == "tg":   # analytic field: host numpy
        reg, grid = cases.build_case(cfg)
        state, setup = None, "host placement (cases.build_case)"
    else:                                         # lattice placement on the device
        reg, grid, state = cases.build_case_device(cfg, dev)
        setup = "device placement (cases.build_case_device, csrc/cases.cu)"
    lib = _native.lib(periodic=grid_is_periodic(grid))
    n = reg.particle_count
    d = reg.dim
    nw = int((reg.raw_view("wall") != 0).sum()) if state is None else \
        int((state["wall"] != 0).sum().item())
    nf = n - nw
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(local_rank))
    if state is not None:
        sim.load_device_state(state)
        del state
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    sim.initialize()
    for _ in range(args.warmup):
        sim.advance()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    sampler = ClockSampler(local_rank)
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = lib.sph_kernel_launches()
    sampler.mark_start()
    times, nsubs = [], []
    for _ in range(args.steps):
        flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        sim.advance()
        ev1.record()
        ev1.synchronize()
        times.append(ev0.elapsed_time(ev1) / 1e3)
        nsubs.append(sim.last_nsub)
    torch.cuda.synchronize()
    sampler.mark_end()
    clocks = sampler.stop()
    launches = lib.sph_kernel_launches() - launches0 - 0
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
        total = float(t.item())
    value = world * n * args.steps / total

    # per-kernel pass (untimed for `value`): one more step with CUDA events
    sim.kernel_times = {}
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    sim.advance()
    ev1.record()
    ev1.synchronize()
    prof_step_s = ev0.elapsed_time(ev1) / 1e3
    kt = {k: statistics.mean(v) / 1e3 for k, v in sim.kernel_times.items()}
    sim.kernel_times = None
    nnb = reg.view("nnb")      # last sub-step's neighbour counts (pull)
    wall = reg.view("wall")
    nnb_f = int(nnb[wall == 0].sum())
    nnb_wf = int(nnb[wall != 0].sum())
    dominant = max(kt, key=kt.get)
    peaks, peak_src = measured_peaks()
    bytes_dom = kernel_bytes(dominant, d, nf, nw, nnb_f, 0, nnb_wf)
    achieved = bytes_dom / kt[dominant] / 1e9
    traffic, issue = None, None
    prof_json = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_json):
        with open(prof_json) as fh:
            ent = json.load(fh).get(args.config, {}).get(dominant)
        if isinstance(ent, dict):
            traffic = ent.get("dram_bytes")
            issue = ent.get("issue_active_pct")
            issue = issue / 100.0 if issue is not None else None

    # end-to-end through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(sim, reg, max(1, min(args.steps, 3)), world, dev)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        pus, done, secs, thr, cn = cpu_oracle_run(args.config, 1, args.cpu_budget)
        cpu = {"value": pus, "unit": UNIT, "cores": thr, "kind": "port",
               "sample": f"{done} full advective step(s) (nsub={cn}) of the same "
                         f"case after an untimed initialize(); C port of the "
                         f"reference (oracle/sph_oracle.c, bit-identical), "
                         f"OpenMP {thr} threads"}

    ncells = grid.cell_count
    passes = max(1, math.ceil(max(1, (ncells - 1).bit_length()) / 8))
    b_full = step_bytes_model(d, n, nf, nw, statistics.mean(nsubs), ncells, passes)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (mixed f64)",
        "data": data_label(args.config),
        "config": {"workload": CONFIGS[args.config][0], "case": args.config,
                   "particles": n, "fluid": nf, "wall": nw, "grid_cells": ncells,
                   "nsub_per_step": nsubs, "l2": "flushed between steps (256 MB write)",
                   "parallelism": "single GPU",
                   "setup": f"{setup}, {setup_s:.2f} s (untimed)",
                   "sub_step_updates_per_s": world * n * sum(nsubs) / total},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {
            "bound": "hbm", "kernel": dominant, "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
            "issue_active_frac": issue,
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": bytes_dom,
            "launch_ms": 1e3 * kt[dominant],
            "kernel_ms_per_substep": {k: 1e3 * v for k, v in kt.items()},
            "profiled_step_ms": 1e3 * prof_step_s,
            "step_model_bytes_per_update": b_full,
            "step_model_frac": value / world * b_full / (peaks["hbm_gbs"] * 1e9),
            "note": "the sweeps are instruction-issue bound in bit-exact mode "
                    "(SURVEY 8d): issue_active_frac (ncu smsp__issue_active, "
                    "profiles/ncu_traffic.json) is their binding roof; traffic = "
                    "ncu dram bytes per launch"},
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    if rank == 0:
        emit(line)


def slab_arm(args, rank, world, local_rank):
    """N > 1: the configuration slab-partitioned over the ranks (SURVEY.md
    8e) through distributed.DistributedSimulation with the CUDA engine."""
    import numpy as np
    import torch
    from paper_2603_11868_b200 import _native
    from paper_2603_11868_b200.distributed import (FIELDS, Comm, DistributedSimulation,
                                                   EngineBackend, SlabLayout, cell_plane)
    from paper_2603_11868_b200.physics import force_scalars

    from paper_2603_11868_b200.physics import grid_is_periodic
    dev = torch.device("cuda", local_rank)
    weak = CONFIGS[args.config][1]["kind"] == "tg"   # config 5: fixed work per GPU
    reg, grid = build_case(args.config, world if weak else 1)
    lib = _native.lib(periodic=grid_is_periodic(grid))
    n = reg.particle_count
    d = reg.dim
    nw = int((reg.raw_view("wall") != 0).sum())
    nf = n - nw
    x = reg.raw_view("x")
    planes = cell_plane(x[:, 0], grid.origin.astype(x.dtype)[0], x.dtype.type(grid.cell_size),
                        int(grid.shape[0]))
    layout = SlabLayout.balanced(np.bincount(planes, minlength=int(grid.shape[0])), world)
    mine = layout.owner(planes) == rank
    owned = {f: reg.raw_view(f)[mine] for f in FIELDS}
    sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
    comm = Comm(dev)
    be = EngineBackend(force_scalars(reg, grid), sing, grid, dev)
    sim = DistributedSimulation(comm, be, grid, owned, sing, layout=layout, rebalance_every=10)
    del reg, owned
    sim.initialize()
    for _ in range(args.warmup):
        sim.advance()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = lib.sph_kernel_launches()
    sampler.mark_start()
    times, nsubs = [], []
    for _ in range(args.steps):
        flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        sim.advance()
        ev1.record()
        ev1.synchronize()
        times.append(ev0.elapsed_time(ev1) / 1e3)
        nsubs.append(sim.last_nsub)
    torch.cuda.synchronize()
    sampler.mark_end()
    clocks = sampler.stop()
    launches = lib.sph_kernel_launches() - launches0
    total = float(comm.allreduce([sum(times)], "max")[0])
    value = n * args.steps / total

    e2e = None
    if not args.no_e2e:   # public API with the owned state in pinned host memory
        cap = {f: int(sim.owned[f].shape[0] * 1.5) + 1024 for f in FIELDS}
        host = {f: torch.empty((cap[f],) + tuple(sim.owned[f].shape[1:]),
                               dtype=sim.owned[f].dtype, pin_memory=True) for f in FIELDS}
        cnt = int(sim.owned["id"].shape[0])
        for f in FIELDS:
            host[f][:cnt].copy_(sim.owned[f])
        ksteps = max(1, min(args.steps, 3))
        torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nb_in = nb_out = 0
        for _ in range(ksteps):
            sim.owned = {f: host[f][:cnt].to(dev, non_blocking=True) for f in FIELDS}
            nb_in = sum(host[f][:cnt].numel() * host[f].element_size() for f in FIELDS)
            sim.advance()
            cnt = int(sim.owned["id"].shape[0])
            for f in FIELDS:
                host[f][:cnt].copy_(sim.owned[f])
            nb_out = sum(host[f][:cnt].numel() * host[f].element_size() for f in FIELDS)
        torch.cuda.synchronize()
        secs = float(comm.allreduce([time.perf_counter() - t0], "max")[0])
        e2e = {"value": n * ksteps / secs, "unit": UNIT,
               "h2d_bytes_per_step": nb_in, "d2h_bytes_per_step": nb_out, "steps": ksteps,
               "timer": "host wall clock, max over ranks, around H2D of the owned "
                        "state + advance + D2H (rank 0's bytes)"}
    peaks, peak_src = measured_peaks()
    ncells = grid.cell_count
    passes = max(1, math.ceil(max(1, (ncells - 1).bit_length()) / 8))
    b_full = step_bytes_model(d, n, nf, nw, statistics.mean(nsubs), ncells, passes)
    per_gpu = value / world * b_full / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": "f32 (mixed f64)", "data": data_label(args.config),
        "config": {"workload": CONFIGS[args.config][0], "case": args.config,
                   "particles": n, "fluid": nf, "wall": nw, "grid_cells": ncells,
                   "nsub_per_step": nsubs, "l2": "flushed between steps (256 MB write)",
                   "parallelism": f"slabs x{world} (axis-0, 2-plane halos, NCCL P2P"
                                  + (", periodic ring)" if weak else ")"),
                   "slab_cuts": [int(c) for c in sim.layout.cuts],
                   "sub_step_updates_per_s": n * sum(nsubs) / total},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {
            "bound": "hbm", "kernel": "whole step (byte model)", "achieved": per_gpu,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": per_gpu / peaks["hbm_gbs"],
            "traffic": None, "peak_source": peak_src,
            "step_model_bytes_per_update": b_full,
            "note": "per-GPU step-level byte model (SURVEY 8d); the per-kernel split "
                    "is measured by the 1-GPU run"},
        "cpu_baseline": None,
        "e2e": e2e,
    }
    if rank == 0:
        emit(line)


def e2e_run(sim, reg, steps, world, dev):
    """Same metric through the public API with host registry arrays in pinned
    memory: every step uploads the registry (push), advances, and reads every
    field back (registry.view -> pull)."""
    import numpy as np
    import torch
    from paper_2603_11868_b200.physics import _ENGINE_FIELDS
    for f in _ENGINE_FIELDS:            # move the registry into pinned memory
        var = reg._discrete[f]
        pinned = torch.empty(var.data.shape,
                             dtype=torch.int32 if var.data.dtype == np.uint32
                             else torch.from_numpy(var.data[:0]).dtype,
                             pin_memory=True).numpy().view(var.data.dtype)
        pinned[...] = reg.view(f)
        var.data = pinned
    sim.host_modified()
    nbytes = sum(reg.raw_view(f).nbytes for f in _ENGINE_FIELDS)
    n = reg.particle_count
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.advance()                     # push (H2D) happens inside: host dirty
        for f in _ENGINE_FIELDS:
            reg.view(f)                   # pull (D2H) of the step's result
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([secs], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        secs = float(t.item())
    return {"value": world * n * steps / secs, "unit": UNIT,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "steps": steps, "timer": "host wall clock around push+advance+pull"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="2d1m")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=60.0)
    ap.add_argument("--slab", action="store_true",
                    help="run the slab-decomposition path even on one rank "
                         "(measures its orchestration overhead)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1 or args.slab:
        global _OUT_FD
        sys.stdout.flush()
        _OUT_FD = os.dup(1)
        os.dup2(2, 1)   # library banners (e.g. "NCCL version") go to stderr
        import torch
        local_rank %= max(1, torch.cuda.device_count())   # ranks sharing a GPU (gloo check)
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL between GPUs; SPH_BENCH_BACKEND=gloo runs the same slab path
        # host-staged (e.g. ranks sharing one GPU to validate it -- not a
        # performance configuration)
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_PORT", "29533")):
            os.environ.setdefault(k, v)
        torch.distributed.init_process_group(os.environ.get("SPH_BENCH_BACKEND", "nccl"))
    try:
        if world > 1 or args.slab:
            slab_arm(args, rank, world, local_rank)
        else:
            gpu_arm(args, rank, world, local_rank)
    finally:
        if world > 1 or args.slab:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

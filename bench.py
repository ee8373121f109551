"""Benchmark: full-time-step particle-updates/s of the WCSPH dam break on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3d4m|2d1m|3d16m|tg8m|2dref]
    python bench.py --impl reference ...      (CPU reference arm)

One "step" = one Simulation.advance (physics.py:489-552): CLL rebuild, the
time-step reductions and nsub acoustic sub-steps, exactly the reference's
work.  value = particles x steps / device time (CUDA events on the engine's
stream, summed over the K timed steps; L2 flushed between steps; max over
ranks).  Default workload: BASELINE config 3 (3D dam break, 4M particles),
the largest single-GPU configuration.  At N > 1 the same configuration is
slab-partitioned over the N GPUs (distributed.py: balanced axis-0 slabs,
2-plane halos, NCCL halo exchange and migration; strong scaling, results
bit-identical to one GPU); ``python bench.py --gpus N`` without a launcher
re-executes itself under torch.distributed.run with N ranks.

Windows.  The state after the W warm-up steps is checkpointed; the K-step
window is then run three times from that checkpoint, each doing the same
work (bitwise-deterministic engine: identical nsub lists, asserted):
  1. `value`  -- device-resident, CUDA events around each step;
  2. roofline -- the same steps with per-kernel CUDA events;
  3. `e2e`    -- through the public API with the registry in pinned host
                 memory: every step uploads the registry (push), advances and
                 reads every field back (pull); host wall clock.

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
DEFAULT_CONFIG = "3d4m"
METRIC = "particle-updates/sec (full time step)"
UNIT = "particle-updates/s"
SUBSTEP_KERNELS = ("kick_drift", "list_filter", "continuity_du", "wall_pressure",
                   "momentum_kick")
L2_NOTE = "flushed between steps (256 MB write > 126 MB L2)"


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


def is_weak(name):
    return CONFIGS[name][1]["kind"] == "tg"


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
    start from it."""
    from paper_2603_11868_b200 import cases
    return cases.build_case(case_config(name, world if is_weak(name) else 1))


def data_label(name):
    if is_weak(name):
        return "synthetic (periodic Taylor-Green lattice, analytic initial field)"
    return "synthetic (reference lattice dam break, deterministic)"


def config_of(name, world, n, nf, nw, ncells):
    """The workload description both arms print (identical dicts)."""
    par = "single GPU" if world == 1 else \
        f"slabs x{world} (axis-0, 2-plane halos, NCCL P2P" + (", periodic ring)" if is_weak(name)
                                                               else ")")
    return {"workload": CONFIGS[name][0], "case": name, "particles": int(n),
            "fluid": int(nf), "wall": int(nw), "grid_cells": int(ncells),
            "precision": "f32 run (the reference's mixed f32/f64 arithmetic, bit-exact)",
            "l2": L2_NOTE, "parallelism": par}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, \
            "fallback (B200_PROFILING.md)"


# -- algorithmic bytes -------------------

def kernel_bytes(name, d, n, nf, nw):
    """Compulsory DRAM bytes of one launch by SURVEY.md 8(d)'s model: each
    field the reference's body reads once, each field it writes once (fp32
    run, u32 id/wall); gathered neighbour data cache-resident; neighbour-list
    traffic is implementation overhead, reported separately (list_bytes)."""
    if name == "continuity_du":    # reads x v rho m id wall, writes rho p  (8d+24)
        return nf * (8 * d + 24)
    if name == "momentum_kick":    # reads x v rho p m id wall, writes v x dvdt (20d+20)
        return nf * (20 * d + 20)
    if name == "wall_pressure":    # walls' own x id wall, writes p rho  (4d+16)
        return nw * (4 * d + 16)
    if name == "kick_drift":       # boundary kick1 + drift: reads x v dvdt, writes x v
        return nf * 20 * d
    if name == "cll_rebuild":      # keys (4d+4) + radix passes (16 per pass) + gather
        return n * (4 * d + 4 + 16 * 3)
    return 0                       # list upkeep / skin build: not in the reference's model


def list_bytes(name, nnb_f, nnb_w, skin_f, skin_w):
    """Neighbour-list bytes the implementation streams per launch (4 B per
    entry read): not algorithmic, reported beside `achieved`."""
    if name == "continuity_du":
        return 4 * skin_f
    if name == "momentum_kick":
        return 4 * nnb_f
    if name == "wall_pressure":
        return 4 * skin_w
    return 0


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

def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model


def cpu_oracle_run(name, steps, budget_s, warmup=0, world=1, warm_budget_s=None):
    """Time the oracle port (all host threads) on the same configuration:
    initialize() and ``warmup`` steps untimed (bounded by warm_budget_s),
    then up to ``steps`` advective steps bounded by ``budget_s`` seconds.
    Returns (PU/s, steps_done, seconds, threads, nsubs, warm_done, case)
    with case = (n, nw, ncells)."""
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    from oracle.oracle import OracleSim
    reg, grid = build_case(name, world)
    sim = OracleSim.from_registry(reg, grid)
    sim.initialize()
    t0 = time.perf_counter()
    warm = 0
    for _ in range(warmup):
        if warm_budget_s is not None and time.perf_counter() - t0 > warm_budget_s:
            break
        sim.advance()
        warm += 1
    n = reg.particle_count
    case = (n, int((reg.raw_view("wall") != 0).sum()), grid.cell_count)
    del reg
    done, total = 0, 0.0
    nsubs = []
    while done < steps:
        t0 = time.perf_counter()
        sim.advance()
        total += time.perf_counter() - t0
        done += 1
        nsubs.append(int(sim.last_nsub))
        if total >= budget_s:
            break
    return (n * done / total, done, total, int(os.environ["OMP_NUM_THREADS"]), nsubs, warm,
            case)


def reference_arm(args, rank, world):
    """The reference's CPU path on the box's host cores: the C restatement
    of minisph's step (oracle/sph_oracle.c; bit-identical to the reference,
    so it runs the same nsub sequence as the GPU arm), OpenMP over every host
    thread, the same W + K window as the GPU arm."""
    if rank != 0:
        return
    pus, done, secs, thr, nsubs, warm, (n, nw, ncells) = cpu_oracle_run(
        args.config, max(1, args.steps), budget_s=args.cpu_budget, warmup=args.warmup,
        world=world)
    line = {
        "impl": "reference", "metric": METRIC, "value": pus, "unit": UNIT,
        "n_gpus": world, "steps": done, "warmup": warm,
        "ms_per_step": 1e3 * secs / done, "higher_is_better": True,
        "scaling": "weak" if is_weak(args.config) else "strong", "vs_baseline": None,
        "dtype": "f32 (mixed f64)", "data": data_label(args.config),
        "config": config_of(args.config, world, n, n - nw, nw, ncells),
        "nsub_per_step": nsubs,
        "cpu_baseline": {
            "value": pus, "unit": UNIT, "cores": thr, "kind": "port",
            "cpu": cpu_info(),
            "sample": f"steps {warm + 1}..{warm + done} of the same case ({done} timed "
                      f"advective steps, nsub={nsubs}) after an untimed initialize() + "
                      f"{warm} warm-up steps; C port of the reference "
                      f"(oracle/sph_oracle.c, bit-identical), OpenMP {thr} threads"},
        "e2e": {"value": pus, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


# -- GPU arm --------------------------------------------------------------------

def checkpoint(sim, reg):
    """Host copy of the registry after a pull + the driver's counters
    (the engine is deterministic: a restored run repeats the same bits)."""
    from paper_2603_11868_b200.physics import _ENGINE_FIELDS
    arrays = {f: reg.view(f).copy() for f in _ENGINE_FIELDS}
    attrs = {k: getattr(sim, k) for k in ("step_count", "time", "interaction_count",
                                          "out_of_bounds", "_skin_factor", "_epoch_backoff",
                                          "_last_step")}
    sim._epoch = None   # the re-push below invalidates the lists: a fresh epoch
    few = int(sim._dev["E"].few_refreshes)
    return arrays, attrs, few


def restore(sim, reg, ck, pinned=None):
    """Registry arrays <- checkpoint (into pinned buffers when given); the
    next advance pushes them (host authoritative)."""
    arrays, attrs, few = ck
    for f, a in arrays.items():
        var = reg._discrete[f]
        if pinned is not None:
            var.data = pinned[f]
        var.data[...] = a
    for k, v in attrs.items():
        setattr(sim, k, v)
    sim._epoch = None
    sim._dev["E"].few_refreshes = few
    sim.host_modified()


def pinned_like(arrays):
    import numpy as np
    import torch
    out = {}
    for f, a in arrays.items():
        t = torch.empty(a.shape, dtype=torch.int32 if a.dtype == np.uint32
                        else torch.from_numpy(a[:0]).dtype, pin_memory=True)
        out[f] = t.numpy().view(a.dtype)
    return out


def state_digest(fields):
    """SHA-256 over x, v, rho, p, drho, dvdt, nnb ordered by particle id
    (`--digest`: 1-rank and N-rank runs of a window must agree)."""
    import hashlib
    import numpy as np
    order = np.argsort(fields["id"], kind="stable")
    h = hashlib.sha256()
    for f in ("x", "v", "rho", "p", "drho", "dvdt", "nnb"):
        h.update(np.ascontiguousarray(fields[f][order]).tobytes())
    return h.hexdigest()


def timed_window(sim, steps, flush, stream, sampler=None):
    """K steps, CUDA events on the engine stream around each, L2 flushed
    between steps; returns (seconds, nsubs)."""
    import torch
    times, nsubs = [], []
    sim.list_modes = []
    if sampler is not None:
        sampler.mark_start()
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        sim.advance()
        ev1.record(stream)
        ev1.synchronize()
        times.append(ev0.elapsed_time(ev1) / 1e3)
        nsubs.append(sim.last_nsub)
        sim.list_modes.append(getattr(sim, "last_list_mode", None))
    torch.cuda.synchronize()
    if sampler is not None:
        sampler.mark_end()
    return sum(times), nsubs


def gpu_arm(args, rank, world, local_rank):
    import numpy as np
    import torch
    from paper_2603_11868_b200 import ExecutionPolicy, _native
    from paper_2603_11868_b200.physics import Simulation, grid_is_periodic, _ENGINE_FIELDS
    from paper_2603_11868_b200 import cases

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = case_config(args.config)
    t_setup = time.perf_counter()
    if is_weak(args.config):   # analytic field: host numpy
        reg, grid = cases.build_case(cfg)
        state, setup = None, "host placement (cases.build_case)"
    else:                      # lattice placement on the device
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
    stream = sim._dev["tstream"]
    ck = checkpoint(sim, reg)                 # after W steps (untimed)
    sim._ensure_device()                      # re-push, untimed
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    # 1. value: device-resident window
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.cuda.synchronize()
    launches0 = lib.sph_kernel_launches()
    total, nsubs = timed_window(sim, args.steps, flush, stream, sampler)
    clocks = sampler.stop()
    launches = lib.sph_kernel_launches() - launches0
    value = n * args.steps / total
    interactions_end = sim.interaction_count
    list_modes = list(sim.list_modes)
    digest = state_digest({f: reg.view(f) for f in _ENGINE_FIELDS}) if args.digest else None

    # 2. roofline: the same window with per-kernel CUDA events
    restore(sim, reg, ck)
    sim._ensure_device()
    sim.kernel_times = {}
    total_k, nsubs_k = timed_window(sim, args.steps, flush, stream)
    kt_ms = {k: statistics.mean(v) for k, v in sim.kernel_times.items()}
    sim.kernel_times = None
    assert nsubs_k == nsubs and sim.interaction_count == interactions_end, \
        "kernel-timed window diverged from the value window"
    # neighbour and skin entries of the last sub-step (lists after the window)
    nnb = reg.view("nnb")
    wallv = reg.view("wall")
    nnb_f = int(nnb[wallv == 0].sum())
    nnb_w = int(nnb[wallv != 0].sum())
    skin_f, skin_w = sim.skin_entries()

    # 3. e2e: the same window through the public API, registry in pinned memory
    e2e = None
    if not args.no_e2e:
        pinned = pinned_like(ck[0])
        # one untimed round trip first (the path's first use of the pinned
        # registry and of the push's copy stream), then the window from the
        # checkpoint again
        restore(sim, reg, ck, pinned)
        sim.advance()
        for f in _ENGINE_FIELDS:
            reg.view(f)
        restore(sim, reg, ck, pinned)
        nbytes = sum(reg.raw_view(f).nbytes for f in _ENGINE_FIELDS)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nsubs_e, h2d, d2h, n_ovl, n_pull = [], 0, 0, 0, 0
        trace = os.environ.get("SPH_BENCH_TRACE") == "1"
        for _ in range(args.steps):
            ta = time.perf_counter()
            sim.advance()                     # push (H2D) happens inside: host dirty
            h2d += sim.last_push_bytes
            tb = time.perf_counter()
            for f in _ENGINE_FIELDS:
                reg.view(f)                   # pull (D2H) of the step's result
            d2h += sim.last_pull_bytes
            nsubs_e.append(sim.last_nsub)
            n_ovl += int(sim.last_push_overlapped)
            n_pull += int(sim.last_pull_overlapped)
            if trace:
                print(f"e2e step: advance {1e3 * (tb - ta):.2f} ms, views "
                      f"{1e3 * (time.perf_counter() - tb):.2f} ms, overlapped push "
                      f"{sim.last_push_overlapped}", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        assert nsubs_e == nsubs and sim.interaction_count == interactions_end, \
            "e2e window diverged from the value window"
        e2e = {"value": n * args.steps / secs, "unit": UNIT,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "registry_bytes": nbytes,
               "steps": args.steps, "nsub_per_step": nsubs_e,
               "overlapped_push_steps": int(n_ovl),
               "overlapped_pull_steps": int(n_pull),
               "timer": "host wall clock around push (H2D, pinned, every registry field; "
                        "10 of the 13 fields upload behind the step's skin-list build) + "
                        "advance + pull (D2H of every field the step changed, into the "
                        "registry's host arrays; x and rho/p/drho during the last "
                        "momentum sweep once the step's results are viewed every step; "
                        "m, Vol, id, wall, oflow, rho_scratch are not copied back while "
                        "the device provably holds the pushed values) + registry.view of "
                        "every field, same steps as `value` (restored checkpoint, after "
                        "one untimed round trip)"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        pus, done, secs, thr, cn, warm, _ = cpu_oracle_run(
            args.config, max(1, args.steps), args.cpu_sample_s, warmup=args.warmup,
            warm_budget_s=args.cpu_sample_s)
        cpu = {"value": pus, "unit": UNIT, "cores": thr, "kind": "port",
               "cpu": cpu_info(),
               "sample": f"steps {warm + 1}..{warm + done} ({done} advective steps, "
                         f"nsub={cn}) of the same case after an untimed initialize() + "
                         f"{warm} warm-up steps, bounded to ~{args.cpu_sample_s:.0f} s; "
                         f"C port of the reference (oracle/sph_oracle.c, bit-identical), "
                         f"OpenMP {thr} threads"}

    # roofline of the dominant kernel (SURVEY 8d algorithmic bytes)
    peaks, peak_src = measured_peaks()
    per_launch = {k: v for k, v in kt_ms.items()}
    step_ms = {k: v * (statistics.mean(nsubs) if k in SUBSTEP_KERNELS else 1.0)
               for k, v in per_launch.items()}
    dominant = max(step_ms, key=step_ms.get)
    alg = kernel_bytes(dominant, d, n, nf, nw)
    achieved = alg / (per_launch[dominant] / 1e3) / 1e9
    lb = list_bytes(dominant, nnb_f, nnb_w, skin_f, skin_w)
    traffic, issue, prof_src = None, None, None
    prof_json = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_json):
        with open(prof_json) as fh:
            prof = json.load(fh).get(args.config, {})
        ent = prof.get(dominant)
        prof_src = prof.get("_source")
        if isinstance(ent, dict):
            traffic = ent.get("dram_bytes")
            issue = ent.get("issue_active_pct")
            issue = issue / 100.0 if issue is not None else None
    ncells = grid.cell_count
    passes = max(1, math.ceil(max(1, (ncells - 1).bit_length()) / 8))
    b_full = step_bytes_model(d, n, nf, nw, statistics.mean(nsubs), ncells, passes)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak" if is_weak(args.config) else "strong",
        "vs_baseline": None, "dtype": "f32 (mixed f64)",
        "data": data_label(args.config),
        "config": config_of(args.config, world, n, nf, nw, ncells),
        "nsub_per_step": nsubs,
        "interactions_total": int(interactions_end),
        "state_sha256": digest,
        "skin_lists": {"built": list_modes.count("build"),
                       "carried": list_modes.count("maintain"),
                       "note": "steps whose skin lists were rebuilt / carried over from "
                               "the previous step (sph_engine_maintain_lists)"},
        "sub_step_updates_per_s": n * sum(nsubs) / total,
        "setup": f"{setup}, {setup_s:.2f} s (untimed)",
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {
            "bound": "hbm", "kernel": dominant, "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg,
            "algorithmic_model": "SURVEY.md 8(d): continuity nf(8d+24), momentum "
                                 "nf(20d+20), wall nw(4d+16) bytes per launch",
            "list_bytes_per_launch": lb,
            "traffic_over_algorithmic": (traffic / alg) if traffic and alg else None,
            "binding_roof": "instruction issue (bit-exact FP64-class pair arithmetic, "
                            "SURVEY 8d): issue_active_frac",
            "issue_active_frac": issue,
            "ncu_source": f"profiles/{prof_src}" if prof_src else None,
            "launch_ms": per_launch[dominant],
            "kernel_ms_per_launch": per_launch,
            "kernel_ms_per_step": step_ms,
            "kernel_timed_window_ms_per_step": 1e3 * total_k / args.steps,
            "step_model_bytes_per_update": b_full,
            "step_model_frac": value / world * b_full / (peaks["hbm_gbs"] * 1e9),
            "note": "kernel times: CUDA events on the engine stream over a replay of "
                    "the timed window (same steps, same nsub); traffic = ncu "
                    "dram__bytes_read+write per launch of that kernel"},
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    if rank == 0:
        emit(line)
    del np


def slab_arm(args, rank, world, local_rank):
    """N > 1: the configuration slab-partitioned over the ranks (SURVEY.md
    8e) through distributed.DistributedSimulation with the CUDA engine.  Each
    rank places only its own slab (dam break: device lattice, rows of the
    rank's planes; Taylor-Green: the rank's lattice planes on the host)."""
    import numpy as np
    import torch
    from paper_2603_11868_b200 import _native
    from paper_2603_11868_b200.distributed import (FIELDS, Comm, DistributedSimulation,
                                                   EngineBackend, SlabLayout)
    from paper_2603_11868_b200.physics import force_scalars, grid_is_periodic
    from paper_2603_11868_b200 import cases

    dev = torch.device("cuda", local_rank)
    weak = is_weak(args.config)
    cfg = case_config(args.config, world if weak else 1)
    comm = Comm(dev)
    t_setup = time.perf_counter()
    reg, grid, owned = cases.build_slab_case(cfg, rank, world, dev)
    lib = _native.lib(periodic=grid_is_periodic(grid))
    sing = {k: reg.singular(k) for k in ("rho0", "c0", "h", "g")}
    be = EngineBackend(force_scalars(reg, grid), sing, grid, dev)
    planes = be.planes(owned["x"])
    hist = torch.bincount(planes, minlength=int(grid.shape[0])).cpu().numpy()
    layout = SlabLayout.balanced(comm.allreduce_i64(hist), world)
    cnt = comm.allreduce_i64([int(owned["id"].shape[0]),
                              int((owned["wall"] != 0).sum().item())])
    n, nw = int(cnt[0]), int(cnt[1])
    nf = n - nw
    d = reg.dim
    sim = DistributedSimulation(comm, be, grid, owned, sing, layout=layout, rebalance_every=10)
    del owned
    setup_s = time.perf_counter() - t_setup
    sim.initialize()
    for _ in range(args.warmup):
        sim.advance()
    torch.cuda.synchronize()
    ck = sim.checkpoint()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = lib.sph_kernel_launches()
    stream = torch.cuda.current_stream(dev)
    total, nsubs = timed_window(sim, args.steps, flush, stream, sampler)
    clocks = sampler.stop()
    launches = lib.sph_kernel_launches() - launches0
    total = float(comm.allreduce([total], "max")[0])
    value = n * args.steps / total
    interactions_end = sim.interaction_count
    digest = state_digest(sim.gather()) if args.digest else None

    e2e = None
    if not args.no_e2e:   # the same window, owned state through pinned host memory
        sim.restore(ck)
        host, cap = {}, 0
        nb_in = nb_out = 0
        torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nsubs_e = []
        for _ in range(args.steps):
            cnt = int(sim.owned["id"].shape[0])
            if cnt > cap:   # (re)grow the pinned staging buffers
                cap = int(cnt * 1.25) + 1024
                host = {f: torch.empty((cap,) + tuple(sim.owned[f].shape[1:]),
                                       dtype=sim.owned[f].dtype, pin_memory=True)
                        for f in FIELDS}
            for f in FIELDS:
                host[f][:cnt].copy_(sim.owned[f])
            sim.owned = {f: host[f][:cnt].to(dev, non_blocking=True) for f in FIELDS}
            nb_in = sum(host[f][:cnt].numel() * host[f].element_size() for f in FIELDS)
            sim.advance()
            nsubs_e.append(sim.last_nsub)
            cnt = int(sim.owned["id"].shape[0])
            if cnt > cap:
                cap = int(cnt * 1.25) + 1024
                host = {f: torch.empty((cap,) + tuple(sim.owned[f].shape[1:]),
                                       dtype=sim.owned[f].dtype, pin_memory=True)
                        for f in FIELDS}
            for f in FIELDS:
                host[f][:cnt].copy_(sim.owned[f])
            nb_out = sum(host[f][:cnt].numel() * host[f].element_size() for f in FIELDS)
        torch.cuda.synchronize()
        secs = float(comm.allreduce([time.perf_counter() - t0], "max")[0])
        assert nsubs_e == nsubs and sim.interaction_count == interactions_end, \
            "e2e window diverged from the value window"
        e2e = {"value": n * args.steps / secs, "unit": UNIT,
               "h2d_bytes_per_step": nb_in, "d2h_bytes_per_step": nb_out,
               "steps": args.steps, "nsub_per_step": nsubs_e,
               "timer": "host wall clock, max over ranks, around H2D of the owned "
                        "state + advance + D2H (rank 0's bytes), same steps as `value`"}
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
        "config": config_of(args.config, world, n, nf, nw, ncells),
        "nsub_per_step": nsubs,
        "interactions_total": int(interactions_end),
        "state_sha256": digest,
        "slab_cuts": [int(c) for c in sim.layout.cuts],
        "sub_step_updates_per_s": n * sum(nsubs) / total,
        "setup": f"per-rank slab placement (cases.build_slab_case), {setup_s:.2f} s (untimed)",
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
    del np


def respawn(args):
    """`python bench.py --gpus N` without a launcher: run N ranks under
    torch.distributed.run (one process per GPU) and relay rank 0's line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1" if args.impl == "ours" else
                   str(os.cpu_count() or 1))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=1500.0,
                    help="reference arm: cap on the timed CPU seconds (the default "
                         "lets the 3D 4M window run all K steps)")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0,
                    help="GPU arm's cpu_baseline: bounded CPU sample (s)")
    ap.add_argument("--digest", action="store_true",
                    help="add state_sha256 (by-id hash of the state after the timed "
                         "window) to the line: N-rank runs must equal 1-rank runs")
    ap.add_argument("--slab", action="store_true",
                    help="run the slab-decomposition path even on one rank "
                         "(measures its orchestration overhead)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(respawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1 or args.slab:
        global _OUT_FD
        sys.stdout.flush()
        _OUT_FD = os.dup(1)
        os.dup2(2, 1)   # library banners (e.g. "NCCL version") go to stderr
        import torch
        backend = os.environ.get("SPH_BENCH_BACKEND", "nccl")
        ndev = max(1, torch.cuda.device_count())
        if backend == "nccl" and world > ndev:
            sys.exit(f"bench.py: {world} NCCL ranks need {world} GPUs, {ndev} visible "
                     "(SPH_BENCH_BACKEND=gloo runs ranks sharing a GPU, host-staged: "
                     "a correctness configuration, not a performance one)")
        local_rank %= ndev
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_PORT", "29533")):
            os.environ.setdefault(k, v)
        torch.distributed.init_process_group(backend)
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

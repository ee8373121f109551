"""CPU-baseline calibration, run in the BUILD container (it imports the
reference package from /root/reference, which does not exist on the GPU
box): the reference's numba parallel(8) step against the oracle C port
(OpenMP, 8 threads) on the same cases and steps -> profiles/r02/cpu_calibration.txt."""


import os, sys, time
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/repo")
import numpy as np
import minisph
from minisph import cases as rc
from minisph.physics import Simulation as RSim
from minisph.execution import ExecutionPolicy as RPol
def ref_run(cfg_kw, steps, threads):
    cfg = rc.load_config("/root/reference/pkg/src/minisph/data/kleefsman.cfg") if cfg_kw.get("k") else rc.CaseConfig(case="dambreak2d", dp=cfg_kw["dp"], precision="f32")
    if cfg_kw.get("k"):
        cfg.dp = cfg_kw["dp"]; cfg.precision = "f32"
    from minisph import report as rr
    reg, grid = rr.build_case(cfg)
    sim = RSim(reg, grid, RPol.parallel(threads))
    sim.initialize(); sim.advance()   # JIT warm
    t0 = time.perf_counter()
    for _ in range(steps): sim.advance()
    dt = time.perf_counter() - t0
    return reg.particle_count * steps / dt
def port_run(cfg_kw, steps, threads):
    os.environ["OMP_NUM_THREADS"] = str(threads)
    from paper_2603_11868_b200 import cases
    from oracle.oracle import OracleSim
    cfg = cases.kleefsman_config(dp=cfg_kw["dp"], precision="f32") if cfg_kw.get("k") else cases.CaseConfig(case="dambreak2d", dp=cfg_kw["dp"], precision="f32")
    reg, grid = cases.build_case(cfg)
    sim = OracleSim.from_registry(reg, grid); sim.initialize(); sim.advance()
    t0 = time.perf_counter()
    for _ in range(steps): sim.advance()
    return reg.particle_count * steps / (time.perf_counter() - t0)
for name, kw, steps in (("2d dp=0.00288 (250k)", dict(dp=0.00288), 3), ("3d kleefsman dp=0.02 (180k)", dict(k=1, dp=0.02), 3)):
    r = ref_run(kw, steps, 8)
    p = port_run(kw, steps, 8)
    print(f"{name}: numba parallel(8) {r:.4g} PU/s, C port OpenMP 8 {p:.4g} PU/s, port/numba {p/r:.2f}", flush=True)

"""Per-step wall time of the registry round trip (advance with its push +
views that pull) with and without the overlapped push, on a bench case."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from bench import build_case, pinned_like
    from paper_2603_11868_b200 import ExecutionPolicy
    from paper_2603_11868_b200.physics import Simulation, _ENGINE_FIELDS
    reg, grid = build_case(sys.argv[1] if len(sys.argv) > 1 else "3d4m")
    pinned = pinned_like({f: reg.view(f) for f in _ENGINE_FIELDS})
    for f in _ENGINE_FIELDS:
        var = reg._discrete[f]
        pinned[f][...] = var.data
        var.data = pinned[f]
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    for mode in (True, False, True):
        sim.push_overlap = mode
        for k in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sim.advance()
            t1 = time.perf_counter()
            for f in _ENGINE_FIELDS:
                reg.view(f)
            t2 = time.perf_counter()
            print(f"overlap={mode} step {k}: advance {1e3 * (t1 - t0):7.2f} ms  pull "
                  f"{1e3 * (t2 - t1):6.2f} ms  overlapped={sim.last_push_overlapped} "
                  f"nsub={sim.last_nsub}", flush=True)


if __name__ == "__main__":
    main()

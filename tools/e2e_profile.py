"""Where the end-to-end (registry round trip) time goes: push, step, pull."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from bench import build_case
    from paper_2603_11868_b200 import ExecutionPolicy
    from paper_2603_11868_b200.physics import Simulation, _ENGINE_FIELDS
    reg, grid = build_case(sys.argv[1] if len(sys.argv) > 1 else "2d1m")
    sim = Simulation(reg, grid, ExecutionPolicy.cuda(0))
    sim.initialize()
    for f in _ENGINE_FIELDS:
        var = reg._discrete[f]
        pinned = torch.empty(var.data.shape, dtype=torch.int32 if var.data.dtype == np.uint32
                             else torch.from_numpy(var.data[:0]).dtype,
                             pin_memory=True).numpy().view(var.data.dtype)
        pinned[...] = reg.view(f)
        var.data = pinned
    for _ in range(2):
        sim.advance()
    T = {"push": 0.0, "advance_rest": 0.0, "pull": 0.0}
    K = 3
    for _ in range(K):
        sim.host_modified()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim._ensure_device()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sim.advance()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for f in _ENGINE_FIELDS:
            reg.view(f)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        T["push"] += t1 - t0
        T["advance_rest"] += t2 - t1
        T["pull"] += t3 - t2
    for k, v in T.items():
        print(f"{k:14s} {1e3 * v / K:8.2f} ms")


if __name__ == "__main__":
    main()
